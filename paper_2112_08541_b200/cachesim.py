"""Dynamic FIFO feature cache on the B200 (drop-in for gnnio.cachesim).

Same public surface as the reference module (`gnnio/cachesim.py`):
`POLICIES` (:22), `CacheConfig` (:25-39), `CacheEngineState` (:190-194),
`cold_state` (:197-203), `warm_static` (:206-224), `CacheSimReport`
(:227-272), `simulate` (:275-363), `amortized_update_ops` (:366-375),
`compare_policies` (:378-409).

The FIFO policy -- BGL's cache -- runs on the device (`bgl_cache_*`):
per-batch classification against the pre-batch state, insert-after-batch in
ascending ID order, sharded rings (node v on device v % d) plus the shared
host ring. Results (outcome codes, counters, ring contents and tails) are
bit-exact with the reference. The state lives in HBM and persists across
`simulate` calls exactly like the reference's in-place-mutated state.

The static-degree policy -- the paper's comparison baseline (SURVEY.md §8f
"next" #1) -- also runs on the device: `warm_static` selects each shard's
top-degree nodes with a sort-free histogram + ascending compaction and fills
the same rings, lookups use the same kernel and nothing is inserted.
LRU and LFU (the policies the paper compares against and rejects,
PAPER.md:187,333; LruLevel / LfuLevel cachesim.py:110-175) run on the device
too: the same lookup, then one closed-form update per level
(`bgl_cache_update_ordered`, csrc/ordered.cu), bit-exact with the
reference's sequential levels -- so `compare_policies` sweeps all of
`POLICIES` on the GPU. There is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib

POLICIES = ("static-degree", "fifo", "lru", "lfu")
CODE_CHARS = "DPHM"
_POLICY_CODE = {"fifo": 0, "lru": 1, "lfu": 2}


@dataclass
class CacheConfig:
    device_capacity: int
    host_capacity: int = 0
    num_devices: int = 1
    policy: str = "fifo"
    feature_bytes_per_node: int = 512

    def __post_init__(self):
        if self.policy not in POLICIES:
            raise ValueError(f"unknown policy {self.policy!r}; expected one of {POLICIES}")
        if self.num_devices < 1:
            raise ValueError("num_devices must be >= 1")
        if self.device_capacity < 0 or self.host_capacity < 0:
            raise ValueError("capacities must be >= 0")


def _not_on_device(policy: str):
    return NotImplementedError(
        f"policy {policy!r} is not on the B200 path (only BGL's 'fifo' cache is; see SURVEY.md §2)")


class FifoCacheDevice:
    """Owner of one bgl_cache handle (rings, indices, tails, optional rows)."""

    def __init__(self, cfg: CacheConfig, num_nodes: int, row_bytes: int = 0):
        self.cfg = cfg
        self.num_nodes = max(1, int(num_nodes))
        self.row_bytes = int(row_bytes)
        h = _lib.c_vp()
        _lib.check(_lib.load().bgl_cache_create(self.num_nodes, cfg.num_devices, cfg.device_capacity,
                                                cfg.host_capacity, self.row_bytes, _lib.ctypes.byref(h)))
        self.handle = h.value
        self.max_batch = 0
        self.keys = None     # sparse IDs: sorted int64 key of every dense rank (device)
        self.home = None     # sparse IDs: uint8 shard of every dense rank (device)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.load(require_cuda=False).bgl_cache_destroy(h)
            except Exception:
                pass
            self.handle = None

    def reserve(self, num_nodes: int, max_batch: int) -> None:
        lib = _lib.load()
        if num_nodes > self.num_nodes:
            _lib.check(lib.bgl_cache_reserve_nodes(self.handle, int(num_nodes), _lib.stream_ptr()))
            self.num_nodes = int(num_nodes)
        if max_batch > self.max_batch:
            _lib.check(lib.bgl_cache_reserve_batch(self.handle, int(max_batch)))
            self.max_batch = int(max_batch)

    def adopt_keys(self, flat: np.ndarray) -> tuple[torch.Tensor, int]:
        """Sparse node IDs (gnnio's FifoLevel is a dict, cachesim.py:81-107, so
        any int64 ID is valid): run the rings on dense ranks. The key set
        (resident keys + this trace) is deduplicated and sorted on the device by
        the open-addressing hash table (`bgl_hash_unique`); ranks keep the ID
        order, so every ascending insert list is the reference's; resident
        ranks are renamed to their new ranks (`bgl_cache_remap`) and each
        rank's shard is its ID % d (`bgl_cache_set_home_map`). Returns the
        trace's ranks (int32, device) and the dense node-space size."""
        lib = _lib.load()
        st = _lib.stream_ptr()
        new = torch.from_numpy(np.ascontiguousarray(flat, dtype=np.int64)).cuda()
        if self.keys is not None:
            old = self.keys
            old_max = int(self.keys[-1].item()) if self.keys.numel() else 0
        else:                                   # dense ranks so far: their IDs are 0..n-1
            old = torch.arange(self.num_nodes, dtype=torch.int64, device="cuda")
            old_max = self.num_nodes - 1
        allk = torch.cat([old, new])
        n = int(allk.numel())
        key_bits = max(old_max, int(flat.max()) if flat.size else 0).bit_length()
        ws = torch.empty(int(lib.bgl_hash_unique_workspace(n)), dtype=torch.uint8, device="cuda")
        uniq = torch.empty(n, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        rank = torch.empty(n, dtype=torch.int32, device="cuda")
        _lib.check(lib.bgl_hash_unique(allk.data_ptr(), n, key_bits, ws.data_ptr(), uniq.data_ptr(), cnt.data_ptr(),
                                       rank.data_ptr(), st))
        U = int(cnt.item())
        _lib.check(lib.bgl_cache_remap(self.handle, rank.data_ptr(), max(U, 1), st))
        self.num_nodes = max(self.num_nodes, U)
        self.keys = uniq[:U].clone()
        self.home = torch.empty(max(U, 1), dtype=torch.uint8, device="cuda")
        _lib.check(lib.bgl_key_home(self.keys.data_ptr(), None, U, self.cfg.num_devices, self.home.data_ptr(), st))
        _lib.check(lib.bgl_cache_set_home_map(self.handle, self.home.data_ptr()))
        return rank[old.numel():], self.num_nodes

    def rows_ptr(self) -> int:
        return _lib.load().bgl_cache_rows(self.handle) or 0

    def ordered_level(self, level: int):
        """LRU / LFU level `level` (d = the host level): residents in eviction
        order, their LFU freq and tick, the level's tick counter."""
        c = self.cfg
        cap = c.host_capacity if level == c.num_devices else c.device_capacity
        lst = np.zeros(max(cap, 1), dtype=np.int64)
        fq = np.zeros(max(cap, 1), dtype=np.int64)
        tk = np.zeros(max(cap, 1), dtype=np.int64)
        ln = np.zeros(1, dtype=np.int64)
        lt = np.zeros(1, dtype=np.int64)
        md = np.zeros(1, dtype=np.int64)
        _lib.check(_lib.load().bgl_cache_export_ordered(self.handle, level, lst.ctypes.data, ln.ctypes.data,
                                                        fq.ctypes.data, tk.ctypes.data, lt.ctypes.data,
                                                        md.ctypes.data))
        n = int(ln[0])
        lst, fq, tk = lst[:n], fq[:n], tk[:n]
        if self.keys is not None:
            lst = self.keys.cpu().numpy()[lst]
        return lst, fq, tk, int(lt[0]), int(md[0])

    def level_stats(self) -> np.ndarray:
        """int64 [d+1, 2]: cumulative (insertions, evictions) per level, the
        host level last (_Level counters, cachesim.py:45-49)."""
        out = np.zeros((self.cfg.num_devices + 1, 2), dtype=np.int64)
        _lib.check(_lib.load().bgl_cache_level_stats(self.handle, out.ctypes.data))
        return out

    def export(self):
        c = self.cfg
        d, C, Ch = c.num_devices, c.device_capacity, c.host_capacity
        dev_slots = np.full((d, C), -1, dtype=np.int64)
        dev_tails = np.zeros(d, dtype=np.int64)
        host_slots = np.full(Ch, -1, dtype=np.int64)
        host_tail = np.zeros(1, dtype=np.int64)
        _lib.check(_lib.load().bgl_cache_export(self.handle, dev_slots.ctypes.data, dev_tails.ctypes.data,
                                                host_slots.ctypes.data, host_tail.ctypes.data))
        if self.keys is not None:               # dense ranks -> the sparse IDs
            keys = self.keys.cpu().numpy()
            for a in (dev_slots, host_slots):
                m = a >= 0
                a[m] = keys[a[m]]
        return dev_slots, dev_tails, host_slots, int(host_tail[0])


class FifoLevelView:
    """Read-only view of one ring with the FifoLevel attributes the reference
    exposes (`capacity`, `slots`, `tail`, `residency`, `insertions`,
    `evictions`, `metadata_updates`, `__contains__`, `__len__`,
    cachesim.py:42-107). Reading synchronises with the device."""

    def __init__(self, state: "CacheEngineState", level: int):
        self._state = state
        self._level = level

    def _snap(self):
        dev_slots, dev_tails, host_slots, host_tail = self._state.engine.export()
        if self._level < 0:
            return host_slots, host_tail
        return dev_slots[self._level], int(dev_tails[self._level])

    @property
    def capacity(self) -> int:
        c = self._state.cfg
        return c.host_capacity if self._level < 0 else c.device_capacity

    @property
    def slots(self) -> np.ndarray:
        return self._snap()[0]

    @property
    def tail(self) -> int:
        return self._snap()[1]

    def _stat(self, k: int) -> int:
        y = self._state.cfg.num_devices if self._level < 0 else self._level
        return int(self._state.engine.level_stats()[y, k])

    @property
    def insertions(self) -> int:
        """_Level.insertions (cachesim.py:47, incremented at :104)."""
        return 0 if self._state.policy == "static-degree" else self._stat(0)

    @property
    def evictions(self) -> int:
        """_Level.evictions (cachesim.py:48, incremented at :100)."""
        return 0 if self._state.policy == "static-degree" else self._stat(1)

    @property
    def metadata_updates(self) -> int:
        """_Level.metadata_updates (cachesim.py:49): FIFO and static levels
        never update metadata; LRU / LFU count every hit and insert
        (:118-131, :150-174)."""
        if self._state.policy not in ("lru", "lfu"):
            return 0
        return self._ordered()[4]

    def _ordered(self):
        y = self._state.cfg.num_devices if self._level < 0 else self._level
        return self._state.engine.ordered_level(y)

    @property
    def entries(self):
        """LruLevel.entries (cachesim.py:113): residents, least recent first."""
        from collections import OrderedDict
        return OrderedDict((int(v), None) for v in self._ordered()[0])

    @property
    def freq(self) -> dict[int, int]:
        """LfuLevel.freq (cachesim.py:141)."""
        lst, fq, _, _, _ = self._ordered()
        return {int(v): int(f) for v, f in zip(lst, fq)}

    @property
    def tick_of(self) -> dict[int, int]:
        """LfuLevel.tick_of (cachesim.py:142)."""
        lst, _, tk, _, _ = self._ordered()
        return {int(v): int(t) for v, t in zip(lst, tk)}

    @property
    def tick(self) -> int:
        """LfuLevel.tick (cachesim.py:144): ticks handed out so far."""
        return self._ordered()[3]

    @property
    def resident(self) -> frozenset:
        """Resident node set (StaticLevel.resident, cachesim.py:69)."""
        s = self.slots
        return frozenset(int(v) for v in s[s >= 0])

    @property
    def residency(self) -> dict[int, int]:
        s = self.slots
        return {int(v): i for i, v in enumerate(s) if v >= 0}

    def __contains__(self, node) -> bool:
        if self._state.policy in ("lru", "lfu"):
            return bool(np.any(self._ordered()[0] == int(node)))
        return bool(np.any(self.slots == int(node)))

    def __len__(self) -> int:
        if self._state.policy in ("lru", "lfu"):
            return int(self._ordered()[0].size)
        return int(np.count_nonzero(self.slots >= 0))


@dataclass
class CacheEngineState:
    """Device-resident cache state (the reference's CacheEngineState,
    cachesim.py:190-194); `devices[h]` / `host` are views of the rings."""

    cfg: CacheConfig
    engine: FifoCacheDevice
    policy: str = "fifo"

    @property
    def devices(self) -> list[FifoLevelView]:
        return [FifoLevelView(self, h) for h in range(self.cfg.num_devices)]

    @property
    def host(self) -> FifoLevelView:
        return FifoLevelView(self, -1)


def cold_state(cfg: CacheConfig, num_nodes: int = 1, row_bytes: int = 0) -> CacheEngineState:
    """Empty caches (cachesim.py:197-203). The index grows on demand."""
    if cfg.policy == "static-degree":
        raise ValueError("static policy requires warm_static(g, cfg)")
    if cfg.policy not in _POLICY_CODE:
        raise _not_on_device(cfg.policy)
    eng = FifoCacheDevice(cfg, num_nodes, row_bytes)
    if cfg.policy != "fifo":
        _lib.check(_lib.load().bgl_cache_set_policy(eng.handle, _POLICY_CODE[cfg.policy]))
    return CacheEngineState(cfg=cfg, engine=eng, policy=cfg.policy)


def _top_degree(dg, num_shards: int, capacity: int, exclude: torch.Tensor | None):
    """Per shard (v % num_shards) the `capacity` highest-degree nodes, ties to
    the lower ID (np.lexsort((owned, -degs[owned])), cachesim.py:217-218),
    without a sort: degree histogram -> threshold degree t_h and the number
    of degree-t_h nodes still needed; ties ranked by ascending ID.
    Returns (device int32 nodes, shard by shard, each ascending; counts)."""
    lib = _lib.load()
    st = _lib.stream_ptr()
    n, md = dg.num_nodes, max(dg.max_degree, 0)
    xp = None if exclude is None else exclude.data_ptr()
    hist = torch.empty((num_shards, md + 1), dtype=torch.int64, device="cuda")
    _lib.check(lib.bgl_degree_histogram(dg.indptr.data_ptr(), n, num_shards, md, xp, hist.data_ptr(), st))
    h = hist.cpu().numpy()
    thresh = np.full(num_shards, np.iinfo(np.int64).max, dtype=np.int64)   # select nothing
    need = np.zeros(num_shards, dtype=np.int64)
    for s in range(num_shards):
        cum = np.cumsum(h[s][::-1])          # nodes with degree >= md - i
        if capacity <= 0:
            continue
        if capacity >= cum[-1]:
            thresh[s] = -1                   # the whole shard fits
            continue
        i = int(np.searchsorted(cum, capacity))
        thresh[s] = md - i
        need[s] = capacity - (int(cum[i - 1]) if i > 0 else 0)
    th = torch.from_numpy(thresh).cuda()
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")
    ids = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(int(lib.bgl_compact_workspace(n)), dtype=torch.uint8, device="cuda")
    from .distributed import GpuShardOps
    ops = GpuShardOps(num_shards, n, 4)
    tie_sel = torch.zeros(n, dtype=torch.uint8, device="cuda")
    if need.any():
        _lib.check(lib.bgl_select_flags(dg.indptr.data_ptr(), n, num_shards, th.data_ptr(), xp, None, 0,
                                        flags.data_ptr(), st))
        _lib.check(lib.bgl_compact_flags(flags.data_ptr(), n, ids.data_ptr(), cnt.data_ptr(), ws.data_ptr(), st))
        ties = ids[: int(cnt.item())]
        part, _, counts = ops.partition(ties)
        offs = np.concatenate([[0], np.cumsum(counts.cpu().numpy())])
        for s in range(num_shards):
            if need[s]:
                tie_sel[part[offs[s]:offs[s] + need[s]].long()] = 1
    _lib.check(lib.bgl_select_flags(dg.indptr.data_ptr(), n, num_shards, th.data_ptr(), xp, tie_sel.data_ptr(), 1,
                                    flags.data_ptr(), st))
    _lib.check(lib.bgl_compact_flags(flags.data_ptr(), n, ids.data_ptr(), cnt.data_ptr(), ws.data_ptr(), st))
    chosen = ids[: int(cnt.item())]
    part, _, counts = ops.partition(chosen)
    return part.clone(), counts.cpu().numpy().astype(np.int64)


def warm_static(g, cfg: CacheConfig) -> CacheEngineState:
    """Pre-load every device level with the highest-degree nodes it owns and
    the host level with the next-highest-degree nodes (cachesim.py:206-224),
    computed on the device; the levels never change afterwards."""
    if cfg.policy != "static-degree":
        raise ValueError("warm_static requires policy='static-degree'")
    from .graph import device_graph
    dg = device_graph(g)
    d = cfg.num_devices
    dev_nodes, dev_counts = _top_degree(dg, d, cfg.device_capacity, None)
    host_nodes = torch.empty(0, dtype=torch.int32, device="cuda")
    if cfg.host_capacity > 0:
        resident = torch.zeros(dg.num_nodes, dtype=torch.uint8, device="cuda")
        resident[dev_nodes.long()] = 1
        host_nodes, hc = _top_degree(dg, 1, cfg.host_capacity, resident)
    eng = FifoCacheDevice(cfg, dg.num_nodes)
    _lib.check(_lib.load().bgl_cache_warm(eng.handle, dev_nodes.data_ptr(), (_lib.c_i64 * d)(*dev_counts.tolist()),
                                          host_nodes.data_ptr() if host_nodes.numel() else None,
                                          int(host_nodes.numel()), _lib.stream_ptr()))
    return CacheEngineState(cfg=cfg, engine=eng, policy="static-degree")


@dataclass
class CacheSimReport:
    num_devices: int
    feature_bytes_per_node: int
    batch_queries: list[int] = field(default_factory=list)
    batch_own_hits: list[int] = field(default_factory=list)
    batch_peer_hits: list[int] = field(default_factory=list)
    batch_host_hits: list[int] = field(default_factory=list)
    batch_misses: list[int] = field(default_factory=list)
    batch_insertions: list[int] = field(default_factory=list)
    batch_evictions: list[int] = field(default_factory=list)
    batch_metadata_updates: list[int] = field(default_factory=list)
    outcomes: list[list[str]] | None = None

    @property
    def total_queries(self) -> int:
        return sum(self.batch_queries)

    @property
    def device_hits(self) -> int:
        return sum(self.batch_own_hits) + sum(self.batch_peer_hits)

    @property
    def host_hits(self) -> int:
        return sum(self.batch_host_hits)

    @property
    def misses(self) -> int:
        return sum(self.batch_misses)

    @property
    def hit_ratio(self) -> float:
        total = self.total_queries
        return (self.device_hits + self.host_hits) / total if total else 0.0

    @property
    def peer_bytes(self) -> int:
        return sum(self.batch_peer_hits) * self.feature_bytes_per_node

    @property
    def host_to_device_bytes(self) -> int:
        return sum(self.batch_host_hits) * self.feature_bytes_per_node

    @property
    def remote_fetch_bytes(self) -> int:
        return sum(self.batch_misses) * self.feature_bytes_per_node

    @classmethod
    def from_counters(cls, cfg: CacheConfig, counters: np.ndarray, codes=None) -> "CacheSimReport":
        c = np.asarray(counters, dtype=np.int64).reshape(-1, 8)
        rep = cls(num_devices=cfg.num_devices, feature_bytes_per_node=cfg.feature_bytes_per_node,
                  batch_queries=c[:, 0].tolist(), batch_own_hits=c[:, 1].tolist(),
                  batch_peer_hits=c[:, 2].tolist(), batch_host_hits=c[:, 3].tolist(),
                  batch_misses=c[:, 4].tolist(), batch_insertions=c[:, 5].tolist(),
                  batch_evictions=c[:, 6].tolist(), batch_metadata_updates=c[:, 7].tolist())
        if codes is not None:
            lut = np.array(list(CODE_CHARS))
            rep.outcomes = [lut[cd].tolist() for cd in codes]
        return rep


class _UniqueScratch:
    """Bitmap workspace for building sorted distinct insert lists of
    arbitrary (unsorted / duplicated) batches on the device."""

    def __init__(self, num_nodes: int, max_batch: int):
        lib = _lib.load()
        self.n = num_nodes
        self.ws = torch.empty(int(lib.bgl_unique_workspace(num_nodes)), dtype=torch.uint8, device="cuda")
        _lib.call("bgl_unique_workspace_init", self.ws.data_ptr(), num_nodes, _lib.stream_ptr())
        self.uniq = torch.empty(max(max_batch, 1), dtype=torch.int32, device="cuda")
        self.count = torch.zeros(1, dtype=torch.int64, device="cuda")


# dense node-ID space of the direct-address index: beyond it (IDs >= 2^31, or
# an ID space far larger than the trace) the rings run on hash-deduplicated ranks
_DENSE_LIMIT = (1 << 31) - 1


def _sparse_ids(num_nodes: int, total: int) -> bool:
    return num_nodes > _DENSE_LIMIT or num_nodes > max(1 << 26, 16 * total)


def simulate(trace, cfg: CacheConfig, g=None, batch_devices=None, state: CacheEngineState | None = None,
             record_outcomes: bool = False) -> CacheSimReport:
    """Replay an access trace through the two-level multi-device cache
    (cachesim.py:275-363)."""
    static = cfg.policy == "static-degree"
    if static:
        if state is None:
            if g is None:
                raise ValueError("static policy needs the graph for degree warmup")
            state = warm_static(g, cfg)
        elif state.policy != "static-degree":
            raise ValueError("state/policy mismatch")
    elif state is not None and state.policy != cfg.policy:
        raise ValueError("state/policy mismatch")
    if cfg.policy not in POLICIES:
        raise _not_on_device(cfg.policy)
    ordered = cfg.policy in ("lru", "lfu")

    batches = [np.asarray(b, dtype=np.int64).ravel() for b in trace.batches]
    nb = len(batches)
    d = cfg.num_devices
    sizes = np.array([b.size for b in batches], dtype=np.int64)
    flat = np.concatenate(batches) if nb else np.empty(0, np.int64)
    if flat.size and flat.min() < 0:
        raise ValueError("node IDs must be >= 0")
    num_nodes = int(flat.max()) + 1 if flat.size else 1
    sparse = (state is not None and state.engine.keys is not None) or _sparse_ids(num_nodes, flat.size)
    if state is None:
        state = cold_state(cfg, 1 if sparse else num_nodes)
    eng = state.engine
    maxb = int(sizes.max()) if nb else 0
    ids = None
    if sparse and flat.size:
        ids, num_nodes = eng.adopt_keys(flat)
    eng.reserve(num_nodes, maxb)
    counters = torch.zeros((max(nb, 1), 8), dtype=torch.int64, device="cuda")
    if nb == 0:
        return CacheSimReport.from_counters(cfg, np.zeros((0, 8)))

    lib = _lib.load()
    st = _lib.stream_ptr()
    if ids is None:
        ids = torch.from_numpy(flat.astype(np.int32)).cuda()
    offs = np.concatenate([[0], np.cumsum(sizes)])
    # device-side batch lengths (the ABI takes counts on the device)
    lens = torch.from_numpy(sizes).cuda()
    codes = torch.empty(max(flat.size, 1), dtype=torch.uint8, device="cuda") if record_outcomes or ordered else None
    scratch = _UniqueScratch(eng.num_nodes, maxb)
    seg_off = _lib.c_i64 * 1
    c_off = seg_off(0)
    # AccessTrace rows are sorted and distinct (np.unique, sampler.py:157): such a
    # batch is its own insert order, so only other batches need the device unique
    if flat.size:
        inc = np.diff(flat) > 0
        bstart = np.zeros(flat.size, dtype=bool)
        bstart[offs[1:-1][offs[1:-1] < flat.size]] = True
        bad = np.flatnonzero(~inc & ~bstart[1:]) + 1          # positions breaking strict increase in a batch
        unsorted = np.zeros(nb, dtype=bool)
        unsorted[np.searchsorted(offs, bad, side="right") - 1] = True
    else:
        unsorted = np.zeros(nb, dtype=bool)
    if batch_devices is not None:
        bd = np.asarray(batch_devices, dtype=np.int64)
        if bd.size < nb or (nb and (bd[:nb].min() < 0 or bd[:nb].max() >= d)):
            raise ValueError("worker device out of range")
    for i in range(nb):
        worker = int(batch_devices[i]) if batch_devices is not None else i % d
        n = int(sizes[i])
        bptr = ids.data_ptr() + 4 * int(offs[i])
        nptr = lens.data_ptr() + 8 * i
        cptr = counters.data_ptr() + 64 * i
        # sorted distinct set of the batch = the insert order (cachesim.py:341-344)
        if unsorted[i]:
            _lib.check(lib.bgl_unique_sorted(bptr, 1, c_off, nptr, (_lib.c_i64 * 1)(n), eng.num_nodes,
                                             scratch.ws.data_ptr(), scratch.uniq.data_ptr(),
                                             scratch.count.data_ptr(), st))
            sptr, scnt = scratch.uniq.data_ptr(), scratch.count.data_ptr()
        else:
            sptr, scnt = bptr, nptr
        _lib.check(lib.bgl_cache_lookup(eng.handle, bptr, nptr, n, worker, sptr, scnt, n,
                                        None if codes is None else codes.data_ptr() + int(offs[i]),
                                        None, cptr, st))
        if ordered:                            # LRU / LFU: hits reorder / count, then the policy's inserts
            _lib.check(lib.bgl_cache_update_ordered(eng.handle, bptr, nptr, n, codes.data_ptr() + int(offs[i]),
                                                    sptr, cptr, st))
        elif not static:                       # static levels never change (StaticLevel.insert, cachesim.py:74-75)
            _lib.check(lib.bgl_cache_insert(eng.handle, sptr, n, None, cptr, st))
        if unsorted[i]:
            _lib.check(lib.bgl_unique_reset(scratch.ws.data_ptr(), eng.num_nodes, scratch.uniq.data_ptr(),
                                            scratch.count.data_ptr(), n, st))
    host_counters = counters[:nb].cpu().numpy()
    host_codes = None
    if record_outcomes:
        cc = codes.cpu().numpy()
        host_codes = [cc[offs[i]:offs[i + 1]] for i in range(nb)]
    return CacheSimReport.from_counters(cfg, host_counters, host_codes)


def amortized_update_ops(report: CacheSimReport) -> dict[str, float]:
    """Per-batch mean operation counts (cachesim.py:366-375)."""
    nb = max(1, len(report.batch_queries))
    return {
        "lookups_per_batch": report.total_queries / nb,
        "insertions_per_batch": sum(report.batch_insertions) / nb,
        "evictions_per_batch": sum(report.batch_evictions) / nb,
        "metadata_updates_per_batch": sum(report.batch_metadata_updates) / nb,
    }


def compare_policies(g, trace, capacities, policies=POLICIES, num_devices: int = 1, host_capacity: int = 0,
                     feature_bytes_per_node: int = 512) -> list[dict]:
    """Hit-ratio table over a (policy x capacity) sweep (cachesim.py:378-409);
    every cell runs on the device."""
    rows = []
    for policy in policies:
        for cap in capacities:
            cfg = CacheConfig(device_capacity=cap, host_capacity=host_capacity, num_devices=num_devices,
                              policy=policy, feature_bytes_per_node=feature_bytes_per_node)
            rep = simulate(trace, cfg, g=g)
            rows.append({"policy": policy, "capacity": cap, "hit_ratio": rep.hit_ratio,
                         "device_hits": rep.device_hits, "host_hits": rep.host_hits, "misses": rep.misses})
    return rows
