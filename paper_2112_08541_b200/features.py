"""Feature retrieval through BGL's dynamic FIFO cache (net-new API).

The reference never materialises features (`gnnio/graph.py:3-6`); it counts
the bytes a batch would move (`cachesim.py:261-272`). This module adds the
retrieval the paper describes without changing
`simulate`'s signature: `FeatureCacheEngine.state` is a `CacheEngineState`,
so `cachesim.simulate(trace, cfg, state=engine.state)` drives the same
device state, and `retrieve` returns the rows `F[batch]` byte-exactly:

    lookup (pre-batch state) -> gather hits from the HBM ring slots and misses
    from the feature store (pinned host memory read zero-copy over the host
    link, or HBM) -> insert-after-batch, copying each surviving miss's row
    into the slot it lands in.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib
from .cachesim import CacheConfig, CacheEngineState, CacheSimReport, FifoCacheDevice


def synthetic_features(num_nodes: int, dim: int, seed: int = 0, pinned: bool = True,
                       device_resident: bool = False, chunk_rows: int = 1 << 20) -> torch.Tensor:
    """Deterministic float32 table F[v, j] = hash(v, j, seed) (restated in
    oracle/features_oracle.py), generated on the GPU chunk by chunk and
    stored in pinned host memory (or kept in HBM)."""
    if device_resident:
        out = torch.empty((num_nodes, dim), dtype=torch.float32, device="cuda")
        _lib.call("bgl_synthetic_features", 0, num_nodes, dim, seed, out.data_ptr(), _lib.stream_ptr())
        return out
    out = torch.empty((num_nodes, dim), dtype=torch.float32, pin_memory=pinned)
    buf = torch.empty((min(chunk_rows, num_nodes), dim), dtype=torch.float32, device="cuda")
    for lo in range(0, num_nodes, chunk_rows):
        hi = min(num_nodes, lo + chunk_rows)
        _lib.call("bgl_synthetic_features", lo, hi - lo, dim, seed, buf.data_ptr(), _lib.stream_ptr())
        out[lo:hi].copy_(buf[: hi - lo], non_blocking=False)
    return out


def numa_nodes() -> list[int]:
    """Memory NUMA nodes of this host (/sys/devices/system/node)."""
    base = "/sys/devices/system/node"
    try:
        nodes = sorted(int(d[4:]) for d in os.listdir(base) if d.startswith("node") and d[4:].isdigit())
    except OSError:
        return [0]
    return nodes or [0]


def gpu_numa_node(device_index: int) -> int:
    """NUMA node of a GPU's PCIe root (sysfs numa_node of its bus id; 0 when
    the platform reports none)."""
    import subprocess
    try:
        bus = subprocess.run(["nvidia-smi", "-i", str(device_index), "--query-gpu=pci.bus_id",
                              "--format=csv,noheader"], capture_output=True, text=True, timeout=20).stdout.strip()
        dom, rest = bus.split(":", 1)
        path = f"/sys/bus/pci/devices/{dom[-4:].lower()}:{rest.lower()}/numa_node"
        node = int(open(path).read().strip())
        return max(node, 0)
    except Exception:  # noqa: BLE001 -- no nvidia-smi / sysfs entry: one node
        return 0


MPOL_BIND, MPOL_INTERLEAVE = 2, 3


def mbind(addr: int, length: int, mode: int, nodes) -> bool:
    """mbind(2) on [addr, addr + length): the memory policy new pages of the
    range are allocated with (tmpfs mappings keep it as the shared policy of
    the file, so pages faulted by any process follow it). False if the kernel
    refuses (e.g. a container without the syscall)."""
    import ctypes
    import platform
    nr = {"x86_64": 237, "aarch64": 235}.get(platform.machine())
    if nr is None:
        return False
    nodes = list(nodes)
    maxnode = max(nodes) + 2
    words = (maxnode + 63) // 64
    mask = (ctypes.c_ulong * words)()
    for n in nodes:
        mask[n // 64] |= 1 << (n % 64)
    libc = ctypes.CDLL(None, use_errno=True)
    page = os.sysconf("SC_PAGE_SIZE")
    start = addr - addr % page
    rc = libc.syscall(nr, ctypes.c_void_p(start), ctypes.c_ulong(length + (addr - start)), ctypes.c_int(mode),
                      mask, ctypes.c_ulong(maxnode), ctypes.c_uint(0))
    return rc == 0


def feature_store_plan(nbytes: int, local_world: int, gpu_node: int, mode: str | None = None) -> dict:
    """Where the box's shared host feature store lives (multi-GPU):
      * one NUMA node: one /dev/shm copy, no policy;
      * several nodes, room for one copy per GPU node in /dev/shm
        ("replicate", the default): each GPU reads a replica bound to its own
        node, so the N host links' miss reads do not cross the socket link;
      * otherwise ("interleave"): one copy with its pages interleaved over all
        nodes, so the reads spread over every socket's DRAM channels.
    /dev/shm must hold the copies; if not, "private": every process pins its
    own copy (when the RAM allows it; else an error naming the shortfall)."""
    nodes = numa_nodes()
    try:
        st = os.statvfs("/dev/shm")
        shm_free = st.f_bavail * st.f_frsize
    except OSError:
        shm_free = 0
    mode = mode or os.environ.get("BGL_FEATURE_NUMA", "replicate")
    plan = {"numa_nodes": len(nodes), "shm_free_gb": round(shm_free / 1e9, 1), "gpu_node": gpu_node,
            "bytes": nbytes}
    if len(nodes) == 1 or mode == "none":
        plan.update(policy="single", copies=1)
    elif mode == "replicate" and shm_free >= nbytes * len(nodes) * 1.02:
        plan.update(policy="replicate", copies=len(nodes))
    else:
        plan.update(policy="interleave", copies=1)
    if shm_free < nbytes * plan["copies"] * 1.02:
        avail = 0
        try:
            for line in open("/proc/meminfo"):
                if line.startswith("MemAvailable:"):
                    avail = int(line.split()[1]) * 1024
        except OSError:
            pass
        if avail < nbytes * local_world * 1.05:
            raise MemoryError(f"host feature store of {nbytes / 1e9:.1f} GB: /dev/shm has {shm_free / 1e9:.1f} GB free "
                              f"and {local_world} private copies need {nbytes * local_world / 1e9:.1f} GB of "
                              f"{avail / 1e9:.1f} GB available")
        plan.update(policy="private", copies=local_world)
    return plan


def shared_synthetic_features(num_nodes: int, dim: int, seed: int, name: str, local_rank: int, local_world: int,
                              barrier, chunk_rows: int = 1 << 20, numa: str | None = None):
    """One feature store for all GPU processes of a box: a /dev/shm mapping
    (tmpfs) that every process registers as mapped pinned memory
    (bgl_host_register), so the GPUs' miss gathers read the same host copy
    zero-copy (papers100M: 57 GB once, not once per GPU) -- NUMA-aware
    (feature_store_plan): on a multi-socket box one replica per GPU node or
    interleaved pages. The processes fill disjoint chunks; `barrier()` is a
    collective over the box's processes. Returns (features, plan)."""
    numel = num_nodes * dim
    nbytes = numel * 4
    import torch.distributed as dist
    my_node = gpu_numa_node(torch.cuda.current_device())
    plan = feature_store_plan(nbytes, local_world, my_node, numa)
    multi = dist.is_initialized() and local_world > 1
    if multi:                    # every process follows local rank 0's decision
        plans = [None] * dist.get_world_size()
        dist.all_gather_object(plans, plan)
        plan = dict(plans[dist.get_rank() - local_rank], gpu_node=my_node)
    if plan["policy"] == "private":
        t = synthetic_features(num_nodes, dim, seed)
        barrier()
        barrier()
        return t, plan
    nodes = numa_nodes()
    replica = nodes.index(my_node) if plan["policy"] == "replicate" and my_node in nodes else 0
    path = os.path.join("/dev/shm", f"{name}_{replica}")
    # which processes fill which replica: every process fills its own replica's share
    if multi:
        every = [None] * dist.get_world_size()
        dist.all_gather_object(every, replica)
        base = dist.get_rank() - local_rank
        nodes_all = every[base:base + local_world]
    else:
        nodes_all = [replica]
    fillers = [r for r in range(local_world) if nodes_all[r] == replica]
    creator = fillers[0]
    if local_rank == creator:
        t = torch.from_file(path, shared=True, size=numel, dtype=torch.float32)
        if plan["policy"] == "replicate":
            plan["mbind"] = mbind(t.data_ptr(), nbytes, MPOL_BIND, [my_node])
        elif plan["policy"] == "interleave":
            plan["mbind"] = mbind(t.data_ptr(), nbytes, MPOL_INTERLEAVE, nodes)
    barrier()
    if local_rank != creator:
        t = torch.from_file(path, shared=True, size=numel, dtype=torch.float32)
    t = t.view(num_nodes, dim)
    buf = torch.empty((min(chunk_rows, num_nodes), dim), dtype=torch.float32, device="cuda")
    me = fillers.index(local_rank)
    for ci, lo in enumerate(range(0, num_nodes, chunk_rows)):
        if ci % len(fillers) != me:
            continue
        hi = min(num_nodes, lo + chunk_rows)
        _lib.call("bgl_synthetic_features", lo, hi - lo, dim, seed, buf.data_ptr(), _lib.stream_ptr())
        t[lo:hi].copy_(buf[: hi - lo], non_blocking=False)
    _lib.call("bgl_host_register", t.data_ptr(), numel * 4)
    barrier()
    if local_rank == creator:
        os.unlink(path)          # every process holds its mapping; nothing leaks in /dev/shm
    return t, plan


def table_pointer(features: torch.Tensor) -> int:
    """Device-usable pointer of the feature store (HBM or pinned host)."""
    if features.is_cuda:
        return features.data_ptr()
    try:
        return _lib.host_device_pointer(features)      # pinned or registered (mapped) host memory
    except _lib.BGLError:
        raise ValueError("host feature store must be pinned (zero-copy miss path)") from None


class FeatureCacheEngine:
    """Per-batch retrieval through the sharded FIFO cache on one device.

    With `cfg.num_devices = d > 1` the d shards are simulated on this GPU
    (worker of batch i = i % d, as the reference's routing); the multi-GPU
    engine places shard h on GPU h (see pipeline.py).
    """

    def __init__(self, cfg: CacheConfig, features: torch.Tensor, max_batch: int,
                 shard: tuple[int, int] | None = None):
        """shard = (rank, world): this engine is home shard `rank` of a
        node-ID-sharded cache over `world` GPUs (see distributed.py)."""
        if cfg.policy != "fifo":
            raise NotImplementedError("only BGL's FIFO cache runs on the device")
        if features.dim() != 2 or not features.is_contiguous():
            raise ValueError("features must be a contiguous [num_nodes, dim] tensor")
        self.cfg = cfg
        self.features = features
        self.num_nodes, self.dim = features.shape
        self.row_bytes = self.dim * features.element_size()
        self.table = table_pointer(features)
        self.dev = FifoCacheDevice(cfg, self.num_nodes, self.row_bytes)
        self.dev.reserve(self.num_nodes, max_batch)
        if shard is not None:
            if cfg.num_devices != 1:
                raise ValueError("a shard engine holds one device level (num_devices=1)")
            _lib.check(_lib.load().bgl_cache_set_shard(self.dev.handle, int(shard[0]), int(shard[1])))
        self.state = CacheEngineState(cfg=cfg, engine=self.dev, policy="fifo")
        self.max_batch = int(max_batch)
        self.codes = torch.empty(max(max_batch, 1), dtype=torch.uint8, device="cuda")
        self.src_row = torch.empty(max(max_batch, 1), dtype=torch.int64, device="cuda")
        self.n_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.out = torch.empty((max(max_batch, 1), self.dim), dtype=features.dtype, device="cuda")
        self.counters = torch.zeros(8, dtype=torch.int64, device="cuda")
        # host-link miss gather: 74 CTAs x 8 warps saturate the link while
        # leaving half the SMs' load/store pipes to the overlapped sampler
        # (tools/gather_bench.cu, tools/overlap_probe.py)
        self.miss_ctas = int(os.environ.get("BGL_MISS_CTAS", 74))
        self.miss_rows_in_flight = int(os.environ.get("BGL_MISS_ROWS", 2))
        # runs of consecutive IDs as TMA bulk copies (bgl_gather_spans); "0": per-row loads only
        self.miss_spans = os.environ.get("BGL_MISS_SPANS", "1") != "0"

    def _ring_src(self, src_row: torch.Tensor):
        """(ring rows pointer, src_row pointer) for the gathers. A cache of
        device_capacity 0 (allowed by CacheConfig, cachesim.py:38-39) has no
        ring rows and no hits: every row comes from the table, so no src_row
        is passed either."""
        ring = self.dev.rows_ptr() or None
        return ring, (src_row.data_ptr() if ring else None)

    def retrieve_device(self, ids: torch.Tensor, n_dev: torch.Tensor, max_n: int, worker: int,
                        counters: torch.Tensor | None = None, stream=None, out: torch.Tensor | None = None,
                        events=None, codes: torch.Tensor | None = None):
        """Fully device-resident step: ids = sorted distinct int32 node IDs
        (e.g. BatchSampler.uniq) with the live count in n_dev. Rows land in
        `out` (default self.out) in batch order; codes in `codes` (default
        self.codes)."""
        lib = _lib.load()
        st = _lib.stream_ptr(stream)
        cnt = (self.counters if counters is None else counters).data_ptr()
        out = self.out if out is None else out
        codes = self.codes if codes is None else codes
        h = self.dev.handle
        _lib.check(lib.bgl_cache_lookup(h, ids.data_ptr(), n_dev.data_ptr(), max_n, worker, ids.data_ptr(),
                                        n_dev.data_ptr(), max_n, codes.data_ptr(), self.src_row.data_ptr(),
                                        cnt, st))
        if events is not None:
            events[0].record()
        ring, src = self._ring_src(self.src_row)
        if self.features.is_cuda:
            _lib.check(lib.bgl_gather_rows(ids.data_ptr(), src, n_dev.data_ptr(), max_n, ring,
                                           self.table, self.row_bytes, out.data_ptr(), 0, 0, st))
        else:
            # hits from HBM with the whole GPU, then misses over the host link
            # with ~150 warps (keeps the SMs free for the overlapped sampler)
            _lib.check(lib.bgl_gather_rows(ids.data_ptr(), src, n_dev.data_ptr(), max_n, ring,
                                           self.table, self.row_bytes, out.data_ptr(), 1, 0, st))
            _lib.check(lib.bgl_gather_rows(ids.data_ptr(), src, n_dev.data_ptr(), max_n, ring,
                                           self.table, self.row_bytes, out.data_ptr(), 2, self.miss_ctas, st))
        if events is not None:
            events[1].record()
        _lib.check(lib.bgl_cache_insert(h, ids.data_ptr(), max_n, out.data_ptr(), cnt, st))
        if events is not None and len(events) > 2:
            events[2].record()
        return out

    def retrieve_push(self, ids, n_dev, max_n, worker, out, codes, push_rows, push_pos, counters, stream=None):
        """Home-side step of the sharded multi-GPU cache: lookup, gather with
        every row also stored straight into the worker GPU's output at
        push_pos (peer memory, bgl_gather_rows_push), insert-after-batch with
        the ring rows copied from the local `out`."""
        lib = _lib.load()
        st = _lib.stream_ptr(stream)
        h = self.dev.handle
        _lib.check(lib.bgl_cache_lookup(h, ids.data_ptr(), n_dev.data_ptr(), max_n, worker, ids.data_ptr(),
                                        n_dev.data_ptr(), max_n, codes.data_ptr(), self.src_row.data_ptr(),
                                        counters.data_ptr(), st))
        ring, src = self._ring_src(self.src_row)
        passes = [(0, 0)] if self.features.is_cuda else [(1, 0), (2, self.miss_ctas)]
        for mode, ctas in passes:
            _lib.check(lib.bgl_gather_rows_push(ids.data_ptr(), src, n_dev.data_ptr(), max_n,
                                                ring, self.table, self.row_bytes, out.data_ptr(), push_rows,
                                                push_pos.data_ptr(), mode, ctas, st))
        _lib.check(lib.bgl_cache_insert(h, ids.data_ptr(), max_n, out.data_ptr(), counters.data_ptr(), st))

    # -- split form for the software-pipelined step (pipeline.py) ----------------
    def plan_buffers(self):
        """(plan int32 [d, stride, 2], plan_count int64 [d]) for front/back."""
        stride = int(_lib.load().bgl_cache_plan_stride(self.dev.handle, self.max_batch))
        plan = torch.empty((self.cfg.num_devices, stride, 2), dtype=torch.int32, device="cuda")
        return plan, torch.zeros(self.cfg.num_devices, dtype=torch.int64, device="cuda")

    def lookup_insert(self, ids, n_dev, max_n, worker, codes, src_row, plan, plan_count, counters, stream=None,
                      miss_pos=None, miss_count=None):
        """miss_pos/miss_count given (single-shard engines): the lookup also
        writes the compacted list of device-miss positions for miss_gather."""
        lib = _lib.load()
        st = _lib.stream_ptr(stream)
        h = self.dev.handle
        if miss_pos is not None:
            _lib.check(lib.bgl_cache_lookup_misses(h, ids.data_ptr(), n_dev.data_ptr(), max_n, worker,
                                                   codes.data_ptr(), src_row.data_ptr(), counters.data_ptr(),
                                                   miss_pos.data_ptr(), miss_count.data_ptr(), st))
        else:
            _lib.check(lib.bgl_cache_lookup(h, ids.data_ptr(), n_dev.data_ptr(), max_n, worker, ids.data_ptr(),
                                            n_dev.data_ptr(), max_n, codes.data_ptr(), src_row.data_ptr(),
                                            counters.data_ptr(), st))
        _lib.check(lib.bgl_cache_insert_plan(h, ids.data_ptr(), max_n, plan.data_ptr(), plan_count.data_ptr(),
                                             counters.data_ptr(), st))

    def miss_gather(self, ids, n_dev, max_n, out, src_row, stream=None, miss_pos=None, miss_count=None):
        lib = _lib.load()
        st = _lib.stream_ptr(stream)
        ctas = 0 if self.features.is_cuda else self.miss_ctas
        if miss_pos is not None and self.miss_spans and self.row_bytes % 16 == 0:
            _lib.check(lib.bgl_gather_spans(miss_pos.data_ptr(), miss_count.data_ptr(), max_n, ids.data_ptr(),
                                            self.table, self.row_bytes, out.data_ptr(), ctas, st))
            return
        if miss_pos is not None:     # compacted list: every warp keeps real rows in flight
            _lib.check(lib.bgl_gather_list(miss_pos.data_ptr(), miss_count.data_ptr(), max_n, ids.data_ptr(),
                                           self.table, self.row_bytes, out.data_ptr(), None, None,
                                           self.miss_rows_in_flight, ctas, st))
            return
        ring, src = self._ring_src(src_row)
        _lib.check(lib.bgl_gather_rows(ids.data_ptr(), src, n_dev.data_ptr(), max_n, ring, self.table,
                                       self.row_bytes, out.data_ptr(), 2, ctas, st))

    def back(self, ids, n_dev, max_n, out, src_row, plan, plan_count, stream=None, events=None,
             with_misses: bool = False):
        """Hits' rows from the HBM ring (with_misses: every row, misses from
        the HBM-resident table in the same pass), then the survivors' rows
        into the ring (after the hits were read: the same-batch eviction
        hazard)."""
        lib = _lib.load()
        st = _lib.stream_ptr(stream)
        ring, src = self._ring_src(src_row)
        _lib.check(lib.bgl_gather_rows(ids.data_ptr(), src, n_dev.data_ptr(), max_n, ring, self.table,
                                       self.row_bytes, out.data_ptr(), 0 if with_misses else 1, 0, st))
        if events is not None:
            events[0].record()
        if self.dev.rows_ptr():
            _lib.check(lib.bgl_cache_copy_rows(self.dev.handle, plan.data_ptr(), plan_count.data_ptr(), max_n,
                                               out.data_ptr(), st))

    def retrieve(self, batch_ids, batch_index: int):
        """rows = F[batch_ids] for one sorted distinct batch; returns
        (rows [U, dim] on the device, outcome codes uint8 [U])."""
        if isinstance(batch_ids, torch.Tensor):
            ids = batch_ids.to(device="cuda", dtype=torch.int32)
            unsorted = ids.numel() > 1 and not bool((ids[1:] > ids[:-1]).all())
        else:   # host batch (an AccessTrace row): checked on the host, one H2D copy
            b = np.asarray(batch_ids)
            unsorted = b.size > 1 and not bool(np.all(b[1:] > b[:-1]))
            ids = torch.from_numpy(np.ascontiguousarray(b, dtype=np.int32)).to("cuda", non_blocking=True)
        n = int(ids.numel())
        if n > self.max_batch:
            raise ValueError("batch larger than the engine was sized for")
        if unsorted:
            raise ValueError("retrieve expects a sorted, duplicate-free batch (an AccessTrace batch)")
        self.n_dev.fill_(n)
        worker = batch_index % self.cfg.num_devices
        self.retrieve_device(ids, self.n_dev, n, worker)
        return self.out[:n], self.codes[:n]

    def report(self, nbatches: int = 1) -> CacheSimReport:
        """Cumulative counters as a one-row report."""
        return CacheSimReport.from_counters(self.cfg, self.counters.cpu().numpy())
