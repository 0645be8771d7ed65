"""Multi-hop neighbour sampling + dedup on the B200 (drop-in for gnnio.sampler).

Same public surface and semantics as the reference module
(`gnnio/sampler.py`): `SamplingConfig` (:18-29), `AccessTrace` (:32-40),
`EpochCommReport` (:43-58), `sample_batch` (:97-116), `simulate_epoch`
(:119-167), `save_trace` / `load_trace` (:173-186). Results are bit-exact:
each batch's random stream is numpy's `default_rng((cfg.seed, batch_seed))`
replayed on the device (the host hands the kernels the 256-bit PCG64 state),
hops run in `bgl_sample_hop`, the distinct set in `bgl_unique_sorted`.

`BatchSampler` is the device engine: fixed buffers sized for the largest
batch, device-resident counts, no host sync inside a batch.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .graph import DeviceGraph, device_graph


@dataclass
class SamplingConfig:
    """sampler.py:18-29. `rng` (not in the reference): "replay" reproduces
    gnnio's numpy stream bit for bit (the default, the drop-in); "counter"
    draws from Philox4x32-10 with Floyd's algorithm -- k draws per parent
    instead of deg, same distribution (uniform k-subsets), different stream."""
    fanouts: tuple[int, ...] = (15, 10, 5)
    batch_size: int = 1000
    seed: int = 0
    rng: str = "replay"

    def __post_init__(self):
        self.fanouts = tuple(int(f) for f in self.fanouts)
        if len(self.fanouts) == 0:
            raise ValueError("need at least one hop")
        if any(f < 1 for f in self.fanouts):
            raise ValueError("fanouts must be positive")
        if self.rng not in ("replay", "counter"):
            raise ValueError("rng must be 'replay' or 'counter'")


@dataclass
class AccessTrace:
    """Per batch: sorted array of distinct accessed node IDs."""

    batches: list[np.ndarray]

    def total_accesses(self) -> int:
        return sum(len(b) for b in self.batches)


@dataclass
class EpochCommReport:
    local_accesses: int
    remote_accesses: int
    seed_load: np.ndarray
    request_load: np.ndarray
    bytes_remote_features: int = 0

    @property
    def total_accesses(self) -> int:
        return self.local_accesses + self.remote_accesses

    @property
    def remote_fraction(self) -> float:
        total = self.total_accesses
        return self.remote_accesses / total if total else 0.0


# ----------------------------------------------------------------------------- PCG64 streams

def pcg_states(seed: int, batch_seeds) -> np.ndarray:
    """uint64 [nb, 4] (state_hi, state_lo, inc_hi, inc_lo) of
    `np.random.default_rng((seed, b))` for every b (sampler.py:61-62). Only
    SeedSequence hashing happens on the host; the draws are replayed on the
    device."""
    out = np.empty((len(batch_seeds), 4), dtype=np.uint64)
    m64 = (1 << 64) - 1
    for i, b in enumerate(batch_seeds):
        st = np.random.default_rng((seed, int(b))).bit_generator.state["state"]
        s, inc = int(st["state"]), int(st["inc"])
        out[i] = (s >> 64, s & m64, inc >> 64, inc & m64)
    return out


def pcg_tables(states: np.ndarray, stream=None) -> torch.Tensor:
    """Device jump tables uint64 [nb, 241, 4] (bgl_pcg64_tables)."""
    nb = states.shape[0]
    dev_states = torch.from_numpy(states.view(np.int64).copy()).cuda()
    tables = torch.empty((nb, _lib.PCG_TABLE_ROWS, 4), dtype=torch.int64, device="cuda")
    _lib.call("bgl_pcg64_tables", _lib.ptr(dev_states), nb, _lib.ptr(tables), _lib.stream_ptr(stream))
    return tables


def _i64_array(vals):
    return (ctypes.c_int64 * len(vals))(*[int(v) for v in vals])


class BatchSampler:
    """Device engine for one mini-batch: H hops + sorted distinct set.

    Layout in HBM (`nodes`, int32): [seeds | hop 1 | ... | hop H], segment h
    sized for its worst case cap_h = cap_{h-1} * min(fanout_h, max_degree);
    `counts[h]` (device int64) holds the live length of segment h.
    """

    def __init__(self, g, fanouts, max_batch: int, relabel: bool = False, max_ctas: int = 0, rng: str = "replay",
                 frontier_outputs: bool = True):
        """frontier_outputs=False (pipelines that only need the distinct
        set): no parent_idx stores, and the last hop only marks the dedup
        bitmap (its frontier is never read)."""
        self.dg: DeviceGraph = device_graph(g)
        self.frontier_outputs = bool(frontier_outputs) or relabel
        if rng not in ("replay", "counter"):
            raise ValueError("rng must be 'replay' or 'counter'")
        self.rng = rng
        self.max_ctas = int(max_ctas)   # cap on sampler CTAs (0 = whole GPU)
        self.fanouts = tuple(int(f) for f in fanouts)
        self.H = len(self.fanouts)
        if self.H > 7:
            raise ValueError("at most 7 hops")
        md = max(1, self.dg.max_degree)
        # k = min(fanout, deg) <= max_degree, so clamping is exact and keeps
        # the wide-k path within its 4096 cap.
        self.eff = [min(f, md) for f in self.fanouts]
        caps = [int(max_batch)]
        for f in self.eff:
            caps.append(caps[-1] * f)
        self.caps = caps
        self.seg_off = [0]
        for c in caps:
            self.seg_off.append(self.seg_off[-1] + c)
        total = self.seg_off[-1]
        dev = self.dg.indptr.device
        self.nodes = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
        self.pidx = [torch.empty(max(caps[h + 1], 1), dtype=torch.int32, device=dev) for h in range(self.H)]
        self.counts = torch.zeros(self.H + 1, dtype=torch.int64, device=dev)
        self.draw_base = torch.zeros(self.H + 1, dtype=torch.int64, device=dev)   # [0] stays 0
        lib = _lib.load()
        ws = (lib.bgl_sample_hop_counter_workspace if rng == "counter" else lib.bgl_sample_hop_workspace)
        self.hop_ws = torch.empty(int(ws(max(caps[:-1]))), dtype=torch.uint8, device=dev)
        if rng == "counter" and max(self.eff) > 32:
            raise ValueError("counter-RNG sampler: fanouts must be <= 32")
        n = self.dg.num_nodes
        self.max_uniq = min(total, n)
        self.uws = torch.empty(int(lib.bgl_unique_workspace(n)), dtype=torch.uint8, device=dev)
        _lib.call("bgl_unique_workspace_init", _lib.ptr(self.uws), n, _lib.stream_ptr())
        self.uniq = torch.empty(max(self.max_uniq, 1), dtype=torch.int32, device=dev)
        self.num_uniq = torch.zeros(1, dtype=torch.int64, device=dev)
        self.local = torch.empty(max(total, 1), dtype=torch.int32, device=dev) if relabel else None
        self._c_seg_off = _i64_array(self.seg_off[:-1])
        self._c_seg_max = _i64_array(self.caps)
        self._seg_bytes = [o * 4 for o in self.seg_off]

    @property
    def seeds(self) -> torch.Tensor:
        return self.nodes[: self.caps[0]]

    def load_seeds(self, seeds: torch.Tensor, stream=None) -> None:
        """Copy int32 seeds (device or pinned host) into segment 0."""
        b = seeds.numel()
        if b == 0:
            raise ValueError("seeds must be nonempty")
        if b > self.caps[0]:
            raise ValueError("batch larger than the sampler was sized for")
        self.nodes[:b].copy_(seeds, non_blocking=True)
        self.counts[0].fill_(b)

    def run(self, table: torch.Tensor | int, stream=None, hooks=None, hops=None, dedup: bool = True) -> None:
        """Sample all hops and build the distinct set for the seeds already in
        segment 0. `table` is the batch's PCG64 jump table (241x4 uint64).
        `hops` (a range) / `dedup` run a part of it (software pipelining:
        hops 0..H-2 of one batch beside the last hop of another)."""
        lib = _lib.load()
        st = _lib.stream_ptr(stream)
        tptr = table if isinstance(table, int) else table.data_ptr()
        base = self.nodes.data_ptr()
        cnt = self.counts.data_ptr()
        db = self.draw_base.data_ptr()
        for h in (range(self.H) if hops is None else hops):
            out_ids = base + self._seg_bytes[h + 1]
            out_pidx = self.pidx[h].data_ptr()
            if not self.frontier_outputs:
                out_pidx = None
                if h == self.H - 1:
                    out_ids = None
            if self.rng == "counter":
                _lib.check(lib.bgl_sample_hop_counter(
                    self.dg.indptr.data_ptr(), self.dg.indices.data_ptr(), base + self._seg_bytes[h], cnt + 8 * h,
                    self.caps[h], self.eff[h], tptr, h, out_ids, out_pidx,
                    cnt + 8 * (h + 1), self.hop_ws.data_ptr(), self.uws.data_ptr(), st))
                if hooks is not None:
                    hooks(h)
                continue
            _lib.check(lib.bgl_sample_hop(
                self.dg.indptr.data_ptr(), self.dg.indices.data_ptr(),
                base + self._seg_bytes[h], cnt + 8 * h, self.caps[h], self.eff[h], tptr, db + 8 * h,
                out_ids, out_pidx, cnt + 8 * (h + 1),
                self.hop_ws.data_ptr(), self.uws.data_ptr(), self.max_ctas, st))
            if hooks is not None:
                hooks(h)
        if not dedup:
            return
        # hop outputs were marked by the sampler kernels; mark the seeds and emit
        _lib.check(lib.bgl_unique_sorted(
            base, 1, self._c_seg_off, cnt, self._c_seg_max, self.dg.num_nodes,
            self.uws.data_ptr(), self.uniq.data_ptr(), self.num_uniq.data_ptr(), st))
        if self.local is not None:
            _lib.check(lib.bgl_relabel(base, self.H + 1, self._c_seg_off, cnt, self._c_seg_max,
                                       self.dg.num_nodes, self.uws.data_ptr(), self.local.data_ptr(), st))
        _lib.check(lib.bgl_unique_reset(self.uws.data_ptr(), self.dg.num_nodes, self.uniq.data_ptr(),
                                        self.num_uniq.data_ptr(), self.max_uniq, st))

    def clear_marks(self, stream=None) -> None:
        """Zero the dedup bitmap: a batch whose hops ran without their
        dedup (a pipeline reset between the two halves, run(dedup=False))
        leaves its marks behind."""
        _lib.call("bgl_unique_workspace_init", _lib.ptr(self.uws), self.dg.num_nodes, _lib.stream_ptr(stream))

    # host views (synchronising) -------------------------------------------------
    def host_counts(self) -> list[int]:
        return self.counts.cpu().tolist()

    def frontier(self, h: int, counts=None) -> torch.Tensor:
        counts = counts or self.host_counts()
        o = self.seg_off[h + 1]
        return self.nodes[o:o + counts[h + 1]]

    def parent_idx(self, h: int, counts=None) -> torch.Tensor:
        counts = counts or self.host_counts()
        return self.pidx[h][: counts[h + 1]]

    def distinct(self) -> torch.Tensor:
        return self.uniq[: int(self.num_uniq.item())]


_SAMPLERS: dict = {}


def _sampler_for(g, fanouts, batch: int, relabel=False, rng: str = "replay") -> BatchSampler:
    dg = device_graph(g)
    key = (id(dg), tuple(fanouts), relabel, rng)
    s = _SAMPLERS.get(key)
    if s is None or s.dg is not dg or s.caps[0] < batch:
        cap = max(batch, s.caps[0] if s is not None and s.dg is dg else 0)
        s = BatchSampler(dg, fanouts, cap, relabel=relabel, rng=rng)
        if len(_SAMPLERS) > 8:
            _SAMPLERS.clear()
        _SAMPLERS[key] = s
    return s


def _to_i32_device(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.int32)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).astype(np.int32)).cuda()


_TABLES: dict = {}


def _batch_table(seed: int, batch_seed: int) -> torch.Tensor:
    """PCG64 jump table of default_rng((seed, batch_seed)) (sampler.py:61-62),
    built once per (seed, batch) on this device and reused by later calls."""
    key = (int(seed), int(batch_seed), torch.cuda.current_device())
    t = _TABLES.get(key)
    if t is None:
        if len(_TABLES) >= 4096:
            _TABLES.clear()
        t = _TABLES[key] = pcg_tables(pcg_states(seed, [batch_seed]))[0]
    return t


def sample_batch(g, seeds, cfg: SamplingConfig, batch_seed: int = 0):
    """Per-hop frontiers (with duplicates) and the sorted distinct-node set
    (sampler.py:97-116)."""
    seeds = np.asarray(seeds, dtype=np.int64) if not isinstance(seeds, torch.Tensor) else seeds
    if len(seeds) == 0:
        raise ValueError("seeds must be nonempty")
    s = _sampler_for(g, cfg.fanouts, len(seeds), rng=cfg.rng)
    table = _batch_table(cfg.seed, batch_seed)
    s.load_seeds(_to_i32_device(seeds))
    s.run(table)
    counts = s.host_counts()
    frontiers = [s.frontier(h, counts).cpu().numpy().astype(np.int64) for h in range(s.H)]
    distinct = s.distinct().cpu().numpy().astype(np.int64)
    return frontiers, distinct


def sample_batch_relabelled(g, seeds, cfg: SamplingConfig, batch_seed: int = 0):
    """Device-resident batch with the relabelled subgraph: returns
    (distinct int32[U], per-hop (src_local, dst_local) edge lists where hop h
    edge i links local(parent) -> local(sample i)). local = rank in distinct
    (np.unique return_inverse)."""
    if len(seeds) == 0:
        raise ValueError("seeds must be nonempty")
    s = _sampler_for(g, cfg.fanouts, len(seeds), relabel=True, rng=cfg.rng)
    s.load_seeds(_to_i32_device(seeds))
    s.run(_batch_table(cfg.seed, batch_seed))
    counts = s.host_counts()
    edges = []
    for h in range(s.H):
        po, co = s.seg_off[h], s.seg_off[h + 1]
        child = s.local[co:co + counts[h + 1]]
        parent = s.local[po:po + counts[h]][s.pidx[h][: counts[h + 1]].long()]
        edges.append((parent, child))
    return s.distinct(), edges, s


def simulate_epoch(g, p, schedule, cfg: SamplingConfig):
    """One epoch of sampling with partition accounting (sampler.py:119-167)."""
    batches = [np.asarray(b, dtype=np.int64) for b in schedule.batches]
    dg = device_graph(g)
    if p is None:
        part_of = torch.zeros(dg.num_nodes, dtype=torch.int32, device="cuda")
        k = 1
    else:
        part_of = torch.as_tensor(np.asarray(p.part_of, dtype=np.int32)).cuda()
        k = int(p.k)
    seed_load = torch.zeros(k, dtype=torch.int64, device="cuda")
    request_load = torch.zeros(k, dtype=torch.int64, device="cuda")
    local_remote = torch.zeros(2, dtype=torch.int64, device="cuda")
    trace: list[np.ndarray] = []
    if batches:
        for b in batches:
            if len(b) == 0:
                raise ValueError("seeds must be nonempty")
        maxb = max(len(b) for b in batches)
        s = _sampler_for(dg, cfg.fanouts, maxb, rng=cfg.rng)
        tables = pcg_tables(pcg_states(cfg.seed, range(len(batches))))
        flat = np.concatenate(batches)
        offs = np.concatenate([[0], np.cumsum([len(b) for b in batches])])
        flat_dev = _to_i32_device(flat)
        origins = [torch.empty(max(c, 1), dtype=torch.int32, device="cuda") for c in s.caps]
        # the epoch's trace, appended batch by batch on the device: at most
        # min(n, b * (1 + sum of prod fanouts)) distinct IDs per batch
        trace_buf = torch.empty(max(1, len(batches) * s.max_uniq), dtype=torch.int32, device="cuda")
        trace_off = torch.zeros(len(batches) + 1, dtype=torch.int64, device="cuda")
        lib = _lib.load()
        st = _lib.stream_ptr()
        base = s.nodes.data_ptr()
        cnt = s.counts.data_ptr()
        po = part_of.data_ptr()
        for i, b in enumerate(batches):
            s.load_seeds(flat_dev[offs[i]:offs[i + 1]])
            # seed load (sampler.py:139) and seed origins (:142)
            _lib.check(lib.bgl_comm_account(base, cnt, s.caps[0], None, po, k, seed_load.data_ptr(), None, st))
            _lib.check(lib.bgl_take_i32(po, base, cnt, s.caps[0], origins[0].data_ptr(), st))

            def account(h, s=s):
                # lookups of hop h's parents (sampler.py:146-150) happen before
                # its sampling in the reference; the counts are order-free, so
                # they are accounted right after the hop kernel, then origins
                # propagate through parent_idx (sampler.py:153).
                _lib.check(lib.bgl_comm_account(base + s._seg_bytes[h], cnt + 8 * h, s.caps[h],
                                                origins[h].data_ptr(), po, k, request_load.data_ptr(),
                                                local_remote.data_ptr(), st))
                _lib.check(lib.bgl_take_i32(origins[h].data_ptr(), s.pidx[h].data_ptr(), cnt + 8 * (h + 1),
                                            s.caps[h + 1], origins[h + 1].data_ptr(), st))

            s.run(tables[i], hooks=account)
            # the batch's row of the trace stays on the device (no host sync per batch)
            _lib.check(lib.bgl_trace_append(s.uniq.data_ptr(), s.num_uniq.data_ptr(), s.max_uniq,
                                            trace_buf.data_ptr(), trace_off.data_ptr(), i, st))
        off = trace_off.cpu().numpy()
        flat_trace = trace_buf[: int(off[-1])].cpu().numpy().astype(np.int64)
        trace = [flat_trace[off[i]:off[i + 1]] for i in range(len(batches))]
    lr = local_remote.cpu().tolist()
    return (AccessTrace(batches=trace),
            EpochCommReport(local_accesses=int(lr[0]), remote_accesses=int(lr[1]),
                            seed_load=seed_load.cpu().numpy(), request_load=request_load.cpu().numpy()))


# ----------------------------------------------------------------------------- serialization

def save_trace(trace: AccessTrace, path) -> None:
    """One line per batch, space-separated IDs (sampler.py:173-176)."""
    with open(path, "w") as f:
        for batch in trace.batches:
            f.write(" ".join(map(str, np.asarray(batch, dtype=np.int64).tolist())) + "\n")


def load_trace(path) -> AccessTrace:
    batches = []
    with open(path) as f:
        for line in f:
            line = line.strip()
            if line:
                batches.append(np.array(line.split(), dtype=np.int64))
    return AccessTrace(batches=batches)
