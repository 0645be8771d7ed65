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


# -- LRU / LFU levels (cachesim.py:110-175): batch-parallel closed forms -------------
#
# Within a batch the residency is the pre-batch one (inserts come after the
# batch, cachesim.py:341-344); hits only reorder (LRU move_to_end) or count
# (LFU freq += 1). With the level kept as an ordered resident list `log`:
#   LRU: log in recency order. S = [residents not hit] ++ [hit nodes by their
#        LAST hit in the batch] ++ [inserts, ascending]; every insert evicts
#        the front when full, so e = max(0, len0 + M - C) and the new log is
#        S[e:] (a queue keeps its last C entries).
#   LFU: log in insertion-tick order; eviction takes the min (freq, tick).
#        Inserts have key (1, T + j): above every resident with freq 1 (older
#        ticks) and below every resident with freq >= 2, so with A = the
#        freq-1 residents (tick order) the evictions are the first e of
#        A ++ inserts -- except when the level is full at the first insert and
#        holds no freq-1 node: then the first eviction is the global min
#        (freq, tick) resident and the next e - 1 are inserts.
# Counters per level: insertions += M, evictions += e, metadata_updates +=
# hits + M (C == 0: inserts are no-ops, :122, :156).

class OrderedLevel:
    """One LRU or LFU level as the batch-parallel engine keeps it."""

    def __init__(self, policy: str, capacity: int):
        self.policy = policy
        self.capacity = int(capacity)
        self.log: list[int] = []          # LRU: recency order; LFU: tick order
        self.freq: dict[int, int] = {}    # LFU
        self.tick_of: dict[int, int] = {}
        self.tick = 0
        self.insertions = self.evictions = self.metadata_updates = 0

    def __contains__(self, node):
        return node in self.freq if self.policy == "lfu" else node in self._set()

    def _set(self):
        return set(self.log)

    def apply(self, hits_in_order: list[int], inserts_sorted: list[int]):
        C = self.capacity
        self.metadata_updates += len(hits_in_order)
        M = len(inserts_sorted) if C > 0 else 0
        len0 = len(self.log)
        e = max(0, len0 + M - C) if C > 0 else 0
        if self.policy == "lru":
            last = {}
            for i, v in enumerate(hits_in_order):
                last[v] = i
            hit_nodes = [v for v, _ in sorted(last.items(), key=lambda x: x[1])]
            kept = [v for v in self.log if v not in last]
            S = kept + hit_nodes + (list(inserts_sorted) if C > 0 else [])
            self.log = S[e:]
        else:
            for v in hits_in_order:
                self.freq[v] += 1
            if C > 0 and M:
                k0 = max(0, C - len0)
                A = [v for v in self.log if self.freq[v] == 1]
                X = list(inserts_sorted)
                if e >= 1 and k0 == 0 and not A:
                    victim = min(self.log, key=lambda v: (self.freq[v], self.tick_of[v]))
                    gone = {victim} | set(X[:e - 1])
                else:
                    gone = set((A + X)[:e])
                for j, x in enumerate(X):
                    self.freq[x] = 1
                    self.tick_of[x] = self.tick + 1 + j
                self.tick += M
                self.log = [v for v in self.log + X if v not in gone]
                for v in gone:
                    del self.freq[v]
                    del self.tick_of[v]
        self.insertions += M
        self.evictions += e
        self.metadata_updates += M


def simulate_ordered(policy, batches, device_capacity, host_capacity, num_devices, batch_devices=None,
                     state=None):
    """LRU / LFU engine in the batch-parallel form above; same outputs as the
    reference simulate (counters [nb, 8] incl. metadata updates, codes)."""
    d = num_devices
    if state is None:
        state = ([OrderedLevel(policy, device_capacity) for _ in range(d)], OrderedLevel(policy, host_capacity))
    devs, host = state
    counters = np.zeros((len(batches), 8), dtype=np.int64)
    codes_all = []
    tot = lambda a: sum(getattr(lv, a) for lv in devs) + getattr(host, a)  # noqa: E731
    for i, batch in enumerate(batches):
        worker = batch_devices[i] if batch_devices is not None else i % d
        b0 = (tot("insertions"), tot("evictions"), tot("metadata_updates"))
        sets = [set(lv.log) for lv in devs]
        hset = set(host.log)
        codes = np.empty(len(batch), dtype=np.uint8)
        dev_hits = [[] for _ in range(d)]
        host_hits, dm, fm = [], set(), set()
        for j, v in enumerate(batch):
            v = int(v)
            h = v % d
            if v in sets[h]:
                codes[j] = CODE_D if h == worker else CODE_P
                dev_hits[h].append(v)
            elif v in hset:
                codes[j] = CODE_H
                host_hits.append(v)
                dm.add(v)
            else:
                codes[j] = CODE_M
                dm.add(v)
                fm.add(v)
        for h in range(d):
            devs[h].apply(dev_hits[h], sorted(x for x in dm if x % d == h))
        host.apply(host_hits, sorted(fm))
        c = np.bincount(codes, minlength=4)
        b1 = (tot("insertions"), tot("evictions"), tot("metadata_updates"))
        counters[i] = (len(batch), c[0], c[1], c[2], c[3], b1[0] - b0[0], b1[1] - b0[1], b1[2] - b0[2])
        codes_all.append(codes)
    return counters, codes_all, state
