"""CPU restatement of the reference dynamic FIFO feature cache (test oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows `gnnio/cachesim.py`:
  * ring-buffer level: `slots` (-1 = empty), residency map, `tail`; insert is a
    no-op for capacity 0 or an already-resident node, otherwise evicts the
    occupant of `slots[tail]`, writes, advances tail          (cachesim.py:81-107)
  * engine: d device levels (node n lives on n % d) + one shared host level
                                                             (cachesim.py:190-203)
  * simulate: per batch, worker = batch_devices[i] or i % d; every node is
    classified against the pre-batch state as D (own device), P (peer
    device), H (host) or M (miss); after the batch the device-missed nodes
    (ascending) go to their home level and the full misses (ascending) to the
    host level; per-batch counters                       (cachesim.py:275-363)

`FifoEngine` is the literal sequential restatement; `simulate_batched` is the
batch-parallel closed form the CUDA kernels implement.
"""

from __future__ import annotations

import numpy as np

CODE_D, CODE_P, CODE_H, CODE_M = 0, 1, 2, 3
CODE_CHARS = "DPHM"


class FifoRing:
    """One FIFO level (cachesim.py:81-107)."""

    def __init__(self, capacity: int):
        self.capacity = int(capacity)
        self.slots = np.full(self.capacity, -1, dtype=np.int64)
        self.where: dict[int, int] = {}
        self.tail = 0
        self.insertions = 0
        self.evictions = 0

    def __contains__(self, node):
        return node in self.where

    def __len__(self):
        return len(self.where)

    def insert(self, node: int) -> None:
        if self.capacity == 0 or node in self.where:
            return
        victim = int(self.slots[self.tail])
        if victim >= 0:
            self.where.pop(victim)
            self.evictions += 1
        self.slots[self.tail] = node
        self.where[node] = self.tail
        self.tail = (self.tail + 1) % self.capacity
        self.insertions += 1


class FifoEngine:
    """d device rings + a shared host ring (cachesim.py:190-203)."""

    def __init__(self, device_capacity: int, host_capacity: int, num_devices: int):
        self.devices = [FifoRing(device_capacity) for _ in range(num_devices)]
        self.host = FifoRing(host_capacity)

    def _totals(self):
        ins = sum(r.insertions for r in self.devices) + self.host.insertions
        ev = sum(r.evictions for r in self.devices) + self.host.evictions
        return ins, ev

    def run(self, batches, batch_devices=None):
        """Returns (counters [nb, 7] = queries, own, peer, host, miss,
        insertions, evictions; codes list of uint8 arrays)."""
        d = len(self.devices)
        counters = np.zeros((len(batches), 7), dtype=np.int64)
        codes_all = []
        for i, batch in enumerate(batches):
            worker = batch_devices[i] if batch_devices is not None else i % d
            ins0, ev0 = self._totals()
            codes = np.empty(len(batch), dtype=np.uint8)
            dev_missed, full_missed = [], []
            for j, v in enumerate(batch):
                v = int(v)
                home = v % d
                if v in self.devices[home]:
                    codes[j] = CODE_D if home == worker else CODE_P
                elif v in self.host:
                    codes[j] = CODE_H
                    dev_missed.append(v)
                else:
                    codes[j] = CODE_M
                    dev_missed.append(v)
                    full_missed.append(v)
            for v in sorted(dev_missed):
                self.devices[v % d].insert(v)
            for v in sorted(full_missed):
                self.host.insert(v)
            ins1, ev1 = self._totals()
            counts = np.bincount(codes, minlength=4)
            counters[i] = (len(batch), counts[0], counts[1], counts[2], counts[3],
                           ins1 - ins0, ev1 - ev0)
            codes_all.append(codes)
        return counters, codes_all


def _ring_insert_batched(slots, tail, missed):
    """Closed-form insert of an ascending, duplicate-free miss list into one
    ring. Returns (new_tail, insertions, evictions)."""
    cap = slots.size
    m = missed.size
    if cap == 0 or m == 0:
        return tail, 0, 0
    first = min(m, cap)
    pos = (tail + np.arange(first)) % cap
    evicted = int(np.count_nonzero(slots[pos] >= 0)) + max(0, m - cap)
    survivors = np.arange(max(0, m - cap), m)
    slots[(tail + survivors) % cap] = missed[survivors]
    return (tail + m) % cap, m, evicted


def simulate_batched(batches, device_capacity, host_capacity, num_devices,
                     batch_devices=None, dev_slots=None, dev_tails=None,
                     host_slots=None, host_tail=0):
    """Batch-parallel restatement; same outputs as FifoEngine.run plus the
    final ring contents. State arrays are updated in place when given."""
    d = num_devices
    if dev_slots is None:
        dev_slots = np.full((d, device_capacity), -1, dtype=np.int64)
        dev_tails = np.zeros(d, dtype=np.int64)
    if host_slots is None:
        host_slots = np.full(host_capacity, -1, dtype=np.int64)
    counters = np.zeros((len(batches), 7), dtype=np.int64)
    codes_all = []
    for i, batch in enumerate(batches):
        batch = np.asarray(batch, dtype=np.int64)
        worker = batch_devices[i] if batch_devices is not None else i % d
        home = batch % d
        dev_res = np.zeros(batch.size, dtype=bool)
        for h in range(d):
            sel = home == h
            dev_res[sel] = np.isin(batch[sel], dev_slots[h])
        host_res = np.isin(batch, host_slots)
        codes = np.where(dev_res, np.where(home == worker, CODE_D, CODE_P),
                         np.where(host_res, CODE_H, CODE_M)).astype(np.uint8)
        ins = ev = 0
        dm = np.unique(batch[~dev_res])
        for h in range(d):
            t, a, b = _ring_insert_batched(dev_slots[h], int(dev_tails[h]), dm[dm % d == h])
            dev_tails[h] = t
            ins += a
            ev += b
        fm = np.unique(batch[codes == CODE_M])
        host_tail, a, b = _ring_insert_batched(host_slots, int(host_tail), fm)
        ins += a
        ev += b
        counts = np.bincount(codes, minlength=4)
        counters[i] = (batch.size, counts[0], counts[1], counts[2], counts[3], ins, ev)
        codes_all.append(codes)
    return counters, codes_all, (dev_slots, dev_tails, host_slots, host_tail)


# -- static-degree baseline (cachesim.py:64-79, 206-224) ----------------------------

def static_warm(row_offsets, device_capacity, host_capacity, num_devices):
    """Per device the `device_capacity` highest-degree owned nodes (ties to the
    lower ID), then the host level from the rest. Returns (list of device
    arrays, host array), each in selection order."""
    degs = np.diff(np.asarray(row_offsets, dtype=np.int64))
    n = degs.size
    taken = np.zeros(n, dtype=bool)
    dev = []
    for h in range(num_devices):
        owned = np.arange(h, n, num_devices, dtype=np.int64)
        chosen = owned[np.lexsort((owned, -degs[owned]))][:device_capacity]
        taken[chosen] = True
        dev.append(chosen)
    rest = np.flatnonzero(~taken)
    host = rest[np.lexsort((rest, -degs[rest]))][:host_capacity]
    return dev, host


def static_run(batches, dev_sets, host_set, num_devices, batch_devices=None):
    """Lookups only (static levels never change): (counters [nb, 7], codes)."""
    d = num_devices
    dev_member = [set(int(x) for x in s) for s in dev_sets]
    host_member = set(int(x) for x in host_set)
    counters = np.zeros((len(batches), 7), dtype=np.int64)
    codes_all = []
    for i, batch in enumerate(batches):
        worker = batch_devices[i] if batch_devices is not None else i % d
        codes = np.empty(len(batch), dtype=np.uint8)
        for j, v in enumerate(batch):
            v = int(v)
            if v in dev_member[v % d]:
                codes[j] = CODE_D if v % d == worker else CODE_P
            elif v in host_member:
                codes[j] = CODE_H
            else:
                codes[j] = CODE_M
        c = np.bincount(codes, minlength=4)
        counters[i] = (len(batch), c[0], c[1], c[2], c[3], 0, 0)
        codes_all.append(codes)
    return counters, codes_all
