"""Node-ID-sharded FIFO feature cache across GPUs (one process per GPU).

The reference routes every queried node to its home device `v % d`
(cachesim.py:319-320): a hit on the worker's own device is D, on another
device P (peer), and device misses are inserted into their home level after
the batch in ascending ID order (cachesim.py:341-342). The reference only
*simulates* the d devices in one loop; here the d levels are d GPUs:

  round j: rank w samples batch i = j*d + w (batch rng keyed by i, so the
           sampler needs no exchange; worker of batch i is i % d as in
           cachesim.py:309)
    1. partition   stable split of the sorted distinct IDs by home
                   (bgl_partition_by_home) -> d ascending buckets
    2. exchange    bucket sizes + IDs, NCCL all-to-all (the only data the
                   homes need; tiny: U x 4 B per batch)
    3. serve       home h runs the FIFO engine on the buckets it received in
                   worker order w = 0..d-1 == global batch order, so every
                   shard's state machine sees batches exactly as the
                   reference's; hits come from h's HBM ring, misses from the
                   feature store over h's host link, codes D iff w == h
    4. return      rows (+ outcome codes) back to the workers, all-to-all
    5. scatter     rows into batch order (bgl_scatter_rows)

The host level of the reference is a single shared level (cachesim.py:202),
not sharded: `ShardedPipeline(host_capacity=...)` keeps it on one owner GPU,
which is fed every worker's device-missed IDs in batch order and turns the
codes of its hits from M into H (the rows are read from the host feature store
either way, so it is accounting on the side, off the row path). The
all-to-all baseline (`ShardedFeatureCache`) still requires host_capacity == 0.

`ShardedFeatureCache` is written against two small interfaces -- `ops`
(partition / scatter) and `engine` (serve one worker's bucket) -- whose
product implementations are the CUDA kernels below; the CPU gloo tests plug
the test oracle in to check the exchange protocol without GPUs.
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .cachesim import CacheConfig
from .features import FeatureCacheEngine


class GpuShardOps:
    """Partition / scatter on the device (bgl_partition_by_home, bgl_scatter_rows)."""

    def __init__(self, world: int, max_n: int, row_bytes: int):
        self.world = world
        self.row_bytes = row_bytes
        lib = _lib.load()
        self.ws = torch.empty(int(lib.bgl_partition_workspace(max_n, world)), dtype=torch.uint8, device="cuda")
        self.part = torch.empty(max(max_n, 1), dtype=torch.int32, device="cuda")
        self.pos = torch.empty(max(max_n, 1), dtype=torch.int32, device="cuda")
        self.counts = torch.zeros(world, dtype=torch.int64, device="cuda")
        self.n = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.max_n = max_n

    def partition(self, ids: torch.Tensor):
        n = int(ids.numel())
        if n == 0:                      # (an empty tensor's data_ptr is NULL)
            self.counts.zero_()
            return self.part[:0], self.pos[:0], self.counts
        self.n.fill_(n)
        _lib.call("bgl_partition_by_home", ids.data_ptr(), self.n.data_ptr(), n, self.world, self.part.data_ptr(),
                  self.pos.data_ptr(), self.counts.data_ptr(), self.ws.data_ptr(), _lib.stream_ptr())
        return self.part[:n], self.pos[:n], self.counts

    def scatter(self, pos: torch.Tensor, rows: torch.Tensor, out: torch.Tensor) -> None:
        n = int(pos.numel())
        if n == 0:
            return
        self.n.fill_(n)
        _lib.call("bgl_scatter_rows", pos.data_ptr(), self.n.data_ptr(), n, rows.data_ptr(), self.row_bytes,
                  out.data_ptr(), _lib.stream_ptr())


class GpuShardEngine:
    """Home shard `rank` of the sharded FIFO cache on this GPU."""

    def __init__(self, rank: int, world: int, shard_capacity: int, features: torch.Tensor, max_batch: int,
                 feature_bytes_per_node: int | None = None):
        fb = feature_bytes_per_node or features.shape[1] * features.element_size()
        cfg = CacheConfig(device_capacity=shard_capacity, host_capacity=0, num_devices=1,
                          feature_bytes_per_node=fb)
        self.eng = FeatureCacheEngine(cfg, features, max_batch, shard=(rank, world))
        self.counters = torch.zeros(8, dtype=torch.int64, device="cuda")
        self.n = torch.zeros(1, dtype=torch.int64, device="cuda")

    def serve(self, ids: torch.Tensor, worker: int, rows_out: torch.Tensor, codes_out: torch.Tensor) -> None:
        c = int(ids.numel())
        self.n.fill_(c)
        if c == 0:
            return
        self.eng.retrieve_device(ids, self.n, c, worker, counters=self.counters, out=rows_out, codes=codes_out)

    def serve_push(self, ids: torch.Tensor, worker: int, pos: torch.Tensor, peer_rows: int, peer_codes: int,
                   staging_rows: torch.Tensor, staging_codes: torch.Tensor) -> None:
        """Serve worker `worker`'s bucket and push rows + codes straight into
        its output buffers (peer pointers) at `pos`."""
        c = int(ids.numel())
        if c == 0:
            return
        self.n.fill_(c)
        self.eng.retrieve_push(ids, self.n, c, worker, staging_rows, staging_codes, peer_rows, pos, self.counters)
        _lib.call("bgl_scatter_rows", pos.data_ptr(), self.n.data_ptr(), c, staging_codes.data_ptr(), 1, peer_codes,
                  _lib.stream_ptr())


class ShardedFeatureCache:
    """Collective per-round retrieval through the node-ID-sharded cache."""

    def __init__(self, rank: int, world: int, engine, ops, dim: int, dtype=torch.float32, group=None,
                 device=None):
        self.rank, self.world = rank, world
        self.engine, self.ops = engine, ops
        self.dim, self.dtype = dim, dtype
        self.group = group
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())

    def _a2a(self, out, inp, out_splits, in_splits):
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def step(self, ids: torch.Tensor):
        """ids: this rank's batch (sorted distinct int32 IDs on self.device).
        Returns (rows [U, dim], codes uint8 [U]) in batch order. Collective:
        every rank calls it once per round with its own batch."""
        part, pos, counts = self.ops.partition(ids)
        send_counts = counts.to(torch.int64)
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        sc = send_counts.cpu().tolist()
        rc = recv_counts.cpu().tolist()
        recv_ids = torch.empty(sum(rc), dtype=ids.dtype, device=ids.device)
        self._a2a(recv_ids, part.contiguous(), rc, sc)
        send_rows = torch.empty((sum(rc), self.dim), dtype=self.dtype, device=ids.device)
        send_codes = torch.empty(sum(rc), dtype=torch.uint8, device=ids.device)
        off = 0
        for w in range(self.world):           # worker order == global batch order of the round
            c = rc[w]
            self.engine.serve(recv_ids[off:off + c], w, send_rows[off:off + c], send_codes[off:off + c])
            off += c
        rows_back = torch.empty((sum(sc), self.dim), dtype=self.dtype, device=ids.device)
        codes_back = torch.empty(sum(sc), dtype=torch.uint8, device=ids.device)
        self._a2a(rows_back, send_rows, sc, rc)
        self._a2a(codes_back, send_codes, sc, rc)
        rows = torch.empty((int(ids.numel()), self.dim), dtype=self.dtype, device=ids.device)
        codes = torch.empty(int(ids.numel()), dtype=torch.uint8, device=ids.device)
        self.ops.scatter(pos, rows_back, rows)
        codes[pos.long()] = codes_back
        return rows, codes

    def counters(self) -> torch.Tensor:
        """Cache counters summed over all homes (CacheSimReport totals)."""
        c = self.engine.counters.clone()
        dist.all_reduce(c, group=self.group)
        return c


class PeerPushFeatureCache(ShardedFeatureCache):
    """Same protocol with the row exchange fused into the homes' gather: every
    rank exposes its batch output buffers through CUDA IPC; a home gathers a
    worker's rows (HBM ring hits, host-link misses) and stores each row
    directly into that worker's buffer over NVLink (bgl_gather_rows_push), so
    only IDs and positions travel through the collective. `cpu_collectives`
    routes the small ID exchange through host tensors (gloo), which lets the
    whole data path run with several processes on one GPU for testing."""

    def __init__(self, rank: int, world: int, engine: GpuShardEngine, ops: GpuShardOps, dim: int, max_batch: int,
                 group=None, cpu_collectives: bool = False):
        super().__init__(rank, world, engine, ops, dim, group=group)
        self.cpu = cpu_collectives
        self.out_rows = torch.empty((max(max_batch, 1), dim), dtype=torch.float32, device="cuda")
        self.out_codes = torch.empty(max(max_batch, 16), dtype=torch.uint8, device="cuda")
        self.staging_rows = torch.empty_like(self.out_rows)
        self.staging_codes = torch.empty_like(self.out_codes)
        lib = _lib.load()
        mine = []
        for t in (self.out_rows, self.out_codes):
            h = (_lib.ctypes.c_char * 64)()
            off = _lib.c_i64()
            _lib.check(lib.bgl_ipc_get_handle(t.data_ptr(), h, _lib.ctypes.byref(off)))
            mine.append((bytes(h), off.value))
        handles = [None] * world
        dist.all_gather_object(handles, mine, group=group)
        self.peer_rows, self.peer_codes, self._opened = [], [], []
        for w in range(world):
            if w == rank:
                self.peer_rows.append(self.out_rows.data_ptr())
                self.peer_codes.append(self.out_codes.data_ptr())
                continue
            ptrs = []
            for hb, off in handles[w]:
                p = _lib.c_vp()
                _lib.check(lib.bgl_ipc_open_handle(_lib.ctypes.create_string_buffer(hb, 64), _lib.ctypes.byref(p)))
                ptrs.append(p.value + off)
                self._opened.append(p.value)
            self.peer_rows.append(ptrs[0])
            self.peer_codes.append(ptrs[1])

    def close(self) -> None:
        lib = _lib.load()
        for p in self._opened:
            lib.bgl_ipc_close(p)
        self._opened = []

    def _a2a_any(self, out, inp, out_splits, in_splits):
        if self.cpu:
            o = torch.empty(out.shape, dtype=out.dtype)
            dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits, group=self.group)
            out.copy_(o)
        else:
            dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def step(self, ids: torch.Tensor):
        part, pos, counts = self.ops.partition(ids)
        send_counts = counts.to(torch.int64)
        if self.cpu:
            recv_counts = torch.empty(self.world, dtype=torch.int64)
            dist.all_to_all_single(recv_counts, send_counts.cpu(), group=self.group)
        else:
            recv_counts = torch.empty_like(send_counts)
            dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        sc = send_counts.cpu().tolist()
        rc = recv_counts.cpu().tolist()
        recv_ids = torch.empty(sum(rc), dtype=torch.int32, device=ids.device)
        recv_pos = torch.empty(sum(rc), dtype=torch.int32, device=ids.device)
        self._a2a_any(recv_ids, part.contiguous(), rc, sc)
        self._a2a_any(recv_pos, pos.contiguous(), rc, sc)
        off = 0
        for w in range(self.world):           # worker order == global batch order of the round
            c = rc[w]
            # staging is reused per bucket: stream order puts this bucket's ring
            # insert (which reads it) before the next bucket's gather
            self.engine.serve_push(recv_ids[off:off + c], w, recv_pos[off:off + c], self.peer_rows[w],
                                   self.peer_codes[w], self.staging_rows[:c], self.staging_codes[:c])
            off += c
        # every home's pushes into this rank's buffers must have landed
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        n = int(ids.numel())
        return self.out_rows[:n], self.out_codes[:n]


def ipc_map(tensors, rank: int, world: int, group=None) -> list[list[int]]:
    """Exchange CUDA IPC handles of `tensors` (this rank's buffers) and return,
    per tensor, the device address of every rank's copy as mapped in this
    process (own address for rank == self). Collective."""
    lib = _lib.load()
    mine = []
    for t in tensors:
        h = (_lib.ctypes.c_char * 64)()
        off = _lib.c_i64()
        _lib.check(lib.bgl_ipc_get_handle(t.data_ptr(), h, _lib.ctypes.byref(off)))
        mine.append((bytes(h), off.value))
    handles = [None] * world
    dist.all_gather_object(handles, mine, group=group)
    out, opened = [[0] * world for _ in tensors], []
    for w in range(world):
        for k, t in enumerate(tensors):
            if w == rank:
                out[k][w] = t.data_ptr()
                continue
            hb, off = handles[w][k]
            p = _lib.c_vp()
            _lib.check(lib.bgl_ipc_open_handle(_lib.ctypes.create_string_buffer(hb, 64), _lib.ctypes.byref(p)))
            out[k][w] = p.value + off
            opened.append(p.value)
    return out, opened


class ShardedPipeline:
    """Pipelined, host-sync-free rounds of the node-ID-sharded cache; one
    process per GPU (rank = home shard `rank` of `world`, cachesim.py:319-320).

    Round j, rank w = worker of batch i = j*world + w (cachesim.py:309). Its
    stages:
      S(j)   sample the batch (side stream)
      X(j)   bgl_partition_push: bucket h of the sorted distinct IDs
             (ascending = the insert order, cachesim.py:341-342) and the IDs'
             batch positions stored straight into home h's receive area over
             peer memory; then a barrier (NCCL all-reduce of one int -- the
             only collective on the data path)
      LI(j)  at every home, per bucket w in worker order (= global batch
             order, so each shard's FIFO state machine sees the reference's
             batch sequence): lookup vs the pre-bucket state + index insert,
             outcome codes pushed into worker w's buffer
      M(j)   the worker compacts its device-missed positions (codes H/M from
             every home) and fetches those rows over its own host link into
             its output (TMA spans over runs of consecutive IDs)
      B(j)   per bucket: ring hits pushed into worker w's output (peer
             memory), then the survivors' rows into the home's ring slots,
             read from worker w's output (after the hits were read)
      Z(j)   barrier: every home's pushes of round j landed
    Step k enqueues S(k+3), X(k+2), LI(k+2) || M(k+1) || B(k), Z(k): every
    host link streams its worker's misses of round k+1 while round k+2's
    bookkeeping and round k's ring traffic run beside it (the single-GPU pipeline.py schedule,
    with buckets inside each stage). Dependencies point backwards only; the
    LI chain is strictly ordered, so every output equals the reference's.
    Buffers: receive areas, bucket state and outputs by round % 3 (X(k+3)
    is issued after Z(k), the last reader of set k % 3), samplers by round %
    4. The homes keep no row staging: rows are written once, into the
    worker's output; B(j) copies the survivors into the ring from there (a
    peer read of the miss bytes over NVLink). No host synchronisation:
    counts stay on the device and every launch is sized for the worst case.
    Rows of round j are complete after step j (Z(j)) in out_rows[j % 3];
    round j's results (rows, codes, distinct IDs) are valid only until step
    j + 1 is enqueued: that step's LI(j + 3) rewrites the codes of set j % 3
    and its S(j + 4) the sampler slot (j % 4) holding round j's distinct IDs. `barrier` defaults to an NCCL
    all-reduce on the current stream; tests that put several processes on
    one GPU pass a host barrier.
    """

    NR, NSMP = 3, 4        # round sets (receive/bucket state/outputs), samplers

    def __init__(self, rank: int, world: int, dg, fanouts, batch_size: int, order: torch.Tensor, seed: int,
                 shard_capacity: int, features: torch.Tensor, num_batches: int | None = None, group=None,
                 barrier=None, rng: str = "replay", host_capacity: int = 0, batch_devices=None,
                 host_owner: int = 0):
        from .cachesim import FifoCacheDevice
        from .sampler import BatchSampler, pcg_states, pcg_tables
        self.rank, self.world, self.group = rank, world, group
        self.b = int(batch_size)
        self.order = order.to(device="cuda", dtype=torch.int32).contiguous()
        total = int(self.order.numel())
        from .pipeline import check_num_batches
        self.num_batches = check_num_batches(num_batches, total, self.b)
        self.samplers = [BatchSampler(dg, fanouts, self.b, rng=rng, frontier_outputs=False) for _ in range(self.NSMP)]
        maxu = self.maxu = self.samplers[0].max_uniq
        self.dim = features.shape[1]
        self.engine = FeatureCacheEngine(CacheConfig(device_capacity=shard_capacity, host_capacity=0, num_devices=1,
                                                     feature_bytes_per_node=self.dim * features.element_size()),
                                         features, maxu, shard=(rank, world))
        self.rb = self.engine.row_bytes
        self.tables = pcg_tables(pcg_states(seed, range(self.num_batches)))
        dev = torch.device("cuda", torch.cuda.current_device())
        self.batch_counter = torch.zeros(1, dtype=torch.int64, device=dev)    # rounds staged so far
        self.table_stage = [torch.empty((_lib.PCG_TABLE_ROWS, 4), dtype=torch.int64, device=dev)
                            for _ in range(self.NSMP)]
        W, R = world, self.NR
        # receive areas (written by the workers over peer memory), per round set
        self.recv_ids = torch.zeros((R, W, maxu), dtype=torch.int32, device=dev)
        self.recv_pos = torch.zeros((R, W, maxu), dtype=torch.int32, device=dev)
        self.recv_cnt = torch.zeros((R, W), dtype=torch.int64, device=dev)
        # this rank's outputs as a worker (written by the homes), per round set
        self.out_rows = torch.zeros((R, maxu, self.dim), dtype=features.dtype, device=dev)
        self.out_codes = torch.zeros((R, maxu), dtype=torch.uint8, device=dev)
        # home-side per-(round set, bucket) state
        self.codes = torch.empty((R, W, maxu), dtype=torch.uint8, device=dev)
        self.src_row = torch.empty((R, W, maxu), dtype=torch.int64, device=dev)
        self.miss_pos = torch.empty((R, W, maxu), dtype=torch.int32, device=dev)
        self.miss_cnt = torch.zeros((R, W), dtype=torch.int64, device=dev)
        # worker side: this rank's own device-missed batch positions (codes H/M), per round set
        self.wmiss_pos = torch.empty((R, maxu), dtype=torch.int32, device=dev)
        self.wmiss_cnt = torch.zeros(R, dtype=torch.int64, device=dev)
        self.compact_ws = torch.empty(int(_lib.load().bgl_compact_codes_workspace(maxu)), dtype=torch.uint8,
                                      device=dev)
        self.plans = [[self.engine.plan_buffers() for _ in range(W)] for _ in range(R)]
        # batch -> worker routing (cachesim.py:309): round j's batches (j*W + p) % nb, p = 0..W-1, run on
        # batch_devices[...]; each round must use every worker once (one batch per GPU per step)
        self.route = None
        if batch_devices is not None:
            bd = np.asarray(batch_devices, dtype=np.int64)
            if bd.size < self.num_batches or (bd[:self.num_batches] < 0).any() or (bd[:self.num_batches] >= W).any():
                raise ValueError("worker device out of range")
            period = self.num_batches // math.gcd(self.num_batches, W)
            route = np.array([[bd[(j * W + q) % self.num_batches] for q in range(W)] for j in range(period)])
            if any(sorted(r.tolist()) != list(range(W)) for r in route):
                raise ValueError("batch_devices: every round of world consecutive batches must use each GPU once")
            if not all(r.tolist() == list(range(W)) for r in route):
                self.route = route
        # the shared host level (cachesim.py:202): one FIFO level on the owner GPU, fed the workers' device-missed
        # IDs in batch order; its hits turn those rows' codes from M into H (accounting only: H and M rows are
        # both read from the host feature store)
        self.host_capacity, self.host_owner = int(host_capacity), int(host_owner)
        hl = self.host_capacity > 0
        own = hl and rank == host_owner
        self.hl = None
        if own:
            self.hl = FifoCacheDevice(CacheConfig(device_capacity=self.host_capacity, num_devices=1),
                                      dg.num_nodes, 0)
            self.hl.reserve(dg.num_nodes, maxu)
            self.hl_codes = torch.empty(maxu, dtype=torch.uint8, device=dev)
            self.hl_src = torch.empty(maxu, dtype=torch.int64, device=dev)
            self.hl_mpos = torch.empty(maxu, dtype=torch.int32, device=dev)
            self.hl_mcnt = torch.zeros(1, dtype=torch.int64, device=dev)
            self.hl_counters = torch.zeros(8, dtype=torch.int64, device=dev)
        shape = (R, W, maxu) if own else (1,)
        self.hl_ids = torch.zeros(shape, dtype=torch.int32, device=dev)      # owner's receive area
        self.hl_pos = torch.zeros(shape, dtype=torch.int32, device=dev)
        self.hl_cnt = torch.zeros((R, W) if own else (1,), dtype=torch.int64, device=dev)
        self.counters = torch.zeros(8, dtype=torch.int64, device=dev)
        self.part_counts = torch.zeros(W, dtype=torch.int64, device=dev)
        lib = _lib.load()
        self.part_ws = torch.empty(int(lib.bgl_partition_workspace(maxu, W)), dtype=torch.uint8, device=dev)
        ptrs, self._opened = ipc_map([self.recv_ids, self.recv_pos, self.recv_cnt, self.out_rows, self.out_codes,
                                      self.hl_ids, self.hl_pos, self.hl_cnt], rank, world, group)
        rid, rpos, rcnt, orow, ocode, hid, hpos, hcnt = ptrs
        # this rank's slot in the host-level owner's receive area, per round set
        self.hl_dst = [(hid[host_owner] + (r * W + rank) * maxu * 4, hpos[host_owner] + (r * W + rank) * maxu * 4,
                        hcnt[host_owner] + (r * W + rank) * 8) for r in range(R)] if hl else None
        # this rank's slot in every home's receive area, per round set: [R][W] addresses
        slot = [[(r * W + rank) for _ in range(W)] for r in range(R)]
        self.peer_ids = torch.tensor([[rid[h] + slot[r][h] * maxu * 4 for h in range(W)] for r in range(R)],
                                     dtype=torch.int64, device=dev)
        self.peer_pos = torch.tensor([[rpos[h] + slot[r][h] * maxu * 4 for h in range(W)] for r in range(R)],
                                     dtype=torch.int64, device=dev)
        self.peer_cnt = torch.tensor([[rcnt[h] + slot[r][h] * 8 for h in range(W)] for r in range(R)],
                                     dtype=torch.int64, device=dev)
        self.worker_rows, self.worker_codes = orow, ocode     # per worker w: base of its [R] output sets
        self.token = torch.zeros(1, dtype=torch.int32, device=dev)
        self.barrier = barrier if barrier is not None else (lambda: dist.all_reduce(self.token, group=group))
        self.s_sample = torch.cuda.Stream(priority=-1)      # sampling: high priority (pipeline.py)
        self.s_li, self.s_miss, self.s_back = (torch.cuda.Stream() for _ in range(3))
        self.s_result = torch.cuda.Stream()
        self.reported = [torch.cuda.Event() for _ in range(self.NSMP)]   # result hand-off read the sampler
        self._step_events()
        self.k = 0
        self.primed = False
        self._in_graph = False
        self.miss_timing = None      # list -> _M records (start, end, round set) events (eager steps)
        self.back_timing = None      # list -> _B records (start, end) events (eager steps)
        self.graphs: dict = {}
        # per round (our kernels; the two NCCL barrier kernels not counted): stage + hops (sample + heavy)
        # + dedup (mark, emit, reset); partition (count, scan, push); the worker's miss compaction +
        # gather; per bucket: lookup, insert (2), codes push, hit gather, row copy
        per_hop = 1 if rng == "counter" else 2
        self.kernels_per_round = (1 + per_hop * len(fanouts) + 3) + 3 + (2 if W > 1 else 1) + W * 6 + \
            ((1 + (W * 3 + 1 if own else 0)) if hl else 0)
        self.s_hl = torch.cuda.Stream() if own else None
        self.hl_done = torch.cuda.Event() if own else None

    def close(self) -> None:
        lib = _lib.load()
        for p in self._opened:
            lib.bgl_ipc_close(p)
        self._opened = []

    def position(self, j: int, w: int | None = None) -> int:
        """Position (0..world-1) of worker w's batch in round j (w = this rank)."""
        w = self.rank if w is None else w
        if self.route is None:
            return w
        return int(np.flatnonzero(self.route[j % len(self.route)] == w)[0])

    def workers(self, j: int) -> list[int]:
        """Workers of round j's batches in batch order (the order every home
        serves its buckets in: the global batch order of the reference)."""
        if self.route is None:
            return list(range(self.world))
        return [int(w) for w in self.route[j % len(self.route)]]

    def batch_of(self, j: int) -> int:
        return (j * self.world + self.position(j)) % self.num_batches

    # -- stages ------------------------------------------------------------------
    def _S(self, j: int) -> None:
        """Sample round j (batch (j*world + rank) % num_batches, chosen on the
        device by bgl_stage_batch from a counter, so captured steps replay
        every round of the epoch)."""
        slot = j % self.NSMP
        s = self.samplers[slot]
        with torch.cuda.stream(self.s_sample):
            if not self._in_graph:                                    # (a replayed step follows the whole
                self.s_sample.wait_event(self.parted[slot])           # previous step: implicit there)
                self.s_sample.wait_event(self.mdone[slot])
                self.s_sample.wait_event(self.reported[slot])
            _lib.call("bgl_stage_batch", self.order.data_ptr(), self.order.numel(), self.b, self.num_batches,
                      self.tables.data_ptr(), self.batch_counter.data_ptr(), s.nodes.data_ptr(), s.counts.data_ptr(),
                      self.table_stage[slot].data_ptr(), None, None, self.world, self.position(j),
                      _lib.stream_ptr(self.s_sample))
            s.run(self.table_stage[slot], stream=self.s_sample)
            self.sampled[slot].record(self.s_sample)

    def _X(self, j: int) -> None:
        main = torch.cuda.current_stream()
        s = self.samplers[j % self.NSMP]
        r = j % self.NR
        if not self._in_graph:
            main.wait_event(self.sampled[j % self.NSMP])
        _lib.call("bgl_partition_push", s.uniq.data_ptr(), s.num_uniq.data_ptr(), s.max_uniq, self.world,
                  self.peer_ids[r].data_ptr(), self.peer_pos[r].data_ptr(), self.peer_cnt[r].data_ptr(),
                  self.part_counts.data_ptr(), self.part_ws.data_ptr(), _lib.stream_ptr(main))
        self.parted[j % self.NSMP].record(main)
        self.barrier()                                              # round j's IDs at every home
        self.xdone[r].record(main)

    def _LI(self, j: int) -> None:
        r, maxu, h = j % self.NR, self.maxu, self.engine.dev.handle
        lib = _lib.load()
        with torch.cuda.stream(self.s_li):
            st = _lib.stream_ptr(self.s_li)
            self.s_li.wait_event(self.xdone[r])
            for w in self.workers(j):            # batch order of the round
                ids, pos, cnt = self.recv_ids[r, w], self.recv_pos[r, w], self.recv_cnt[r, w:w + 1]
                plan, pcount = self.plans[r][w]
                _lib.check(lib.bgl_cache_lookup_misses(h, ids.data_ptr(), cnt.data_ptr(), maxu, w,
                                                       self.codes[r, w].data_ptr(), self.src_row[r, w].data_ptr(),
                                                       self.counters.data_ptr(), self.miss_pos[r, w].data_ptr(),
                                                       self.miss_cnt[r, w:w + 1].data_ptr(), st))
                _lib.check(lib.bgl_cache_insert_plan(h, ids.data_ptr(), maxu, plan.data_ptr(), pcount.data_ptr(),
                                                     self.counters.data_ptr(), st))
                _lib.check(lib.bgl_scatter_rows(pos.data_ptr(), cnt.data_ptr(), maxu, self.codes[r, w].data_ptr(), 1,
                                                self.worker_codes[w] + r * maxu, st))
                self.li_done[r][w].record(self.s_li)

    def _M(self, j: int) -> None:
        """The worker fetches its own device-missed rows (codes H/M, pushed
        back by every home in LI(j)) from the feature store into its output:
        its sorted distinct IDs keep their runs of consecutive IDs, so runs go
        as TMA spans and the link sees the single-GPU access pattern (a home
        gathering its bucket would read every world-th row only). The homes'
        B(j) copy the survivors into their rings from this output."""
        r, maxu, rb, eng = j % self.NR, self.maxu, self.rb, self.engine
        slot = j % self.NSMP
        s = self.samplers[slot]
        ctas = 0 if eng.features.is_cuda else eng.miss_ctas
        lib = _lib.load()
        timing = self.miss_timing is not None and not self._in_graph
        with torch.cuda.stream(self.s_miss):
            st = _lib.stream_ptr(self.s_miss)
            if timing:   # measurement pass (bench roofline): the compaction + gather between two events
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), r)
                ev[0].record(self.s_miss)
            pos, cnt = self.own_misses(r)
            if self.world > 1:   # (one home: its lookup's compacted list is already the batch's)
                _lib.check(lib.bgl_compact_codes(self.out_codes[r].data_ptr(), s.num_uniq.data_ptr(), maxu, 2,
                                                 pos.data_ptr(), cnt.data_ptr(), self.compact_ws.data_ptr(), st))
            out = self.out_rows[r]
            if eng.miss_spans and rb % 16 == 0:
                _lib.check(lib.bgl_gather_spans(pos.data_ptr(), cnt.data_ptr(), maxu, s.uniq.data_ptr(), eng.table,
                                                rb, out.data_ptr(), ctas, st))
            else:
                _lib.check(lib.bgl_gather_list(pos.data_ptr(), cnt.data_ptr(), maxu, s.uniq.data_ptr(), eng.table,
                                               rb, out.data_ptr(), None, None, eng.miss_rows_in_flight, ctas, st))
            if self.hl_dst is not None:   # device-missed IDs + positions to the host level's owner
                di, dp, dc = self.hl_dst[r]
                _lib.check(lib.bgl_push_pairs(s.uniq.data_ptr(), pos.data_ptr(), cnt.data_ptr(), maxu, di, dp, dc,
                                              st))
            if timing:
                ev[1].record(self.s_miss)
                self.miss_timing.append(ev)
            self.mdone[slot].record(self.s_miss)
            for w in range(self.world):
                self.miss_done[r][w].record(self.s_miss)

    def own_misses(self, r: int):
        """(positions, count) of this worker's device-missed rows of round set r."""
        if self.world == 1:
            return self.miss_pos[r, 0], self.miss_cnt[r, 0:1]
        return self.wmiss_pos[r], self.wmiss_cnt[r:r + 1]

    def _B(self, j: int) -> None:
        r, maxu, rb, eng = j % self.NR, self.maxu, self.rb, self.engine
        h, ring = eng.dev.handle, eng.dev.rows_ptr() or None
        lib = _lib.load()
        timing = self.back_timing is not None and not self._in_graph
        with torch.cuda.stream(self.s_back):
            st = _lib.stream_ptr(self.s_back)
            if timing:   # measurement pass (bench roofline, peer-push rate): the whole B stage
                bev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for wi, w in enumerate(self.workers(j)):   # batch order: a bucket's survivors land before the
                plan, pcount = self.plans[r][w]          # next bucket's hits read the ring
                cnt = self.recv_cnt[r, w:w + 1]
                out_w = self.worker_rows[w] + r * maxu * rb
                if not self._in_graph:
                    self.s_back.wait_event(self.miss_done[r][w])
                if timing and wi == 0:
                    bev[0].record(self.s_back)     # after the first wait: the stage's own time
                _lib.check(lib.bgl_gather_rows_push(self.recv_ids[r, w].data_ptr(),
                                                    self.src_row[r, w].data_ptr() if ring else None,
                                                    cnt.data_ptr(), maxu, ring, eng.table, rb, None, out_w,
                                                    self.recv_pos[r, w].data_ptr(), 1, 0, st))
                if ring:   # survivors' rows into their ring slots, read back from worker w's output
                    _lib.check(lib.bgl_cache_copy_rows_indexed(h, plan.data_ptr(), pcount.data_ptr(), maxu, out_w,
                                                               self.recv_pos[r, w].data_ptr(), st))
            if timing:
                bev[1].record(self.s_back)
                self.back_timing.append(bev)

    def _HL(self, j: int) -> None:
        """Owner of the shared host level: per batch of round j in batch order,
        the worker's device-missed IDs (pushed in M(j)) are looked up in the
        host level (one FIFO level: hits = H, cachesim.py:330-334) and the
        full misses inserted in ascending order (:343-344); the codes go back
        to the worker as H / M at the rows' batch positions."""
        if self.hl is None:
            return
        r, maxu = j % self.NR, self.maxu
        lib = _lib.load()
        h = self.hl.handle
        with torch.cuda.stream(self.s_hl):
            st = _lib.stream_ptr(self.s_hl)
            for w in self.workers(j):
                ids, pos, cnt = self.hl_ids[r, w], self.hl_pos[r, w], self.hl_cnt[r, w:w + 1]
                _lib.check(lib.bgl_cache_lookup_misses(h, ids.data_ptr(), cnt.data_ptr(), maxu, 0,
                                                       self.hl_codes.data_ptr(), self.hl_src.data_ptr(),
                                                       self.hl_counters.data_ptr(), self.hl_mpos.data_ptr(),
                                                       self.hl_mcnt.data_ptr(), st))
                _lib.check(lib.bgl_cache_insert(h, ids.data_ptr(), maxu, None, self.hl_counters.data_ptr(), st))
                _lib.check(lib.bgl_host_level_codes(self.hl_codes.data_ptr(), pos.data_ptr(), cnt.data_ptr(), maxu,
                                                    self.worker_codes[w] + r * maxu, st))
            self.hl_done.record(self.s_hl)
        # fold into the cache counters on the LI stream (its insert kernels update them too)
        with torch.cuda.stream(self.s_li):
            self.s_li.wait_event(self.hl_done)
            _lib.check(lib.bgl_host_level_account(self.hl_counters.data_ptr(), self.counters.data_ptr(),
                                                  _lib.stream_ptr(self.s_li)))

    def prime(self) -> None:
        """Prologue: S(0..2), X(0), LI(0), M(0), X(1), LI(1)."""
        if self.primed:
            return
        for j in range(3):
            self._S(j)
        self._X(0)
        self._LI(0)
        # M(0) reads the codes every home pushed in LI(0): join + barrier first
        main = torch.cuda.current_stream()
        main.wait_stream(self.s_li)
        self.barrier()
        self.s_miss.wait_stream(main)
        self._M(0)
        self._X(1)
        self._LI(1)
        # step 0 runs M(1), which reads the codes every home pushed in LI(1), and
        # B(0), which reads every worker's M(0) rows: join both side streams and
        # put a barrier behind them, as before M(0) (the end-of-step barrier
        # gives the same ordering to every later step)
        main.wait_stream(self.s_li)
        main.wait_stream(self.s_miss)
        self.barrier()
        self.primed = True

    PHASES = 12            # lcm(NR, NSMP): one captured graph per step phase

    def _streams(self):
        return [x for x in (self.s_sample, self.s_li, self.s_miss, self.s_back, self.s_hl) if x is not None]

    def _step_body(self, k: int) -> None:
        main = torch.cuda.current_stream()
        for x in self._streams():                  # fork (graph capture needs it)
            x.wait_stream(main)
        self._S(k + 3)
        self._X(k + 2)
        self._LI(k + 2)
        self._M(k + 1)
        self._B(k)
        self._HL(k)
        for x in self._streams():                  # the step ends when all its work has
            main.wait_stream(x)
        self.barrier()                                              # every home's pushes of round k landed

    def capture(self) -> None:
        """Capture the step of every phase k % 12 in a CUDA graph (with the
        barriers: NCCL collectives are capturable). Cross-step event waits are
        dropped inside the graphs -- replay order already puts each step
        after the whole previous one."""
        if self.route is not None:
            raise ValueError("batch_devices routing runs eager steps: the captured graphs bake in the bucket order")
        self.prime()
        torch.cuda.synchronize()
        saved = self.batch_counter.clone()
        self._in_graph = True
        self._events_captured = True
        try:
            for phase in range(self.PHASES):
                g = torch.cuda.CUDAGraph()
                cs = torch.cuda.Stream()
                cs.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(cs):
                    with torch.cuda.graph(g, stream=cs):
                        self._step_body(phase)
                torch.cuda.current_stream().wait_stream(cs)
                self.graphs[phase] = g
        finally:
            self._in_graph = False
        torch.cuda.synchronize()
        self.batch_counter.copy_(saved)        # capture does not execute; keep the counter exact

    def step(self) -> None:
        """Enqueue step k: S(k+3), X(k+2), LI(k+2) || M(k+1) || B(k), Z(k).
        No host synchronisation; round k's rows are complete afterwards."""
        self.prime()
        k = self.k
        g = self.graphs.get(k % self.PHASES)
        if g is None:
            self._step_body(k)
        else:
            main = torch.cuda.current_stream()
            main.wait_stream(self.s_result)     # result hand-offs outside the graphs (store_result)
            main.wait_stream(self.s_sample)     # e.g. host seeds copied on the sampling stream
            g.replay()
        self.k += 1

    def _step_events(self) -> None:
        """Cross-step events of the eager path (fresh ones after a capture:
        events recorded while capturing belong to the graphs)."""
        R, W = self.NR, self.world
        self.sampled = [torch.cuda.Event() for _ in range(self.NSMP)]
        self.parted = [torch.cuda.Event() for _ in range(self.NSMP)]
        self.mdone = [torch.cuda.Event() for _ in range(self.NSMP)]    # M(j) read sampler j's distinct IDs
        self.xdone = [torch.cuda.Event() for _ in range(R)]
        self.li_done = [[torch.cuda.Event() for _ in range(W)] for _ in range(R)]
        self.miss_done = [[torch.cuda.Event() for _ in range(W)] for _ in range(R)]
        self._events_captured = False

    def step_eager(self) -> None:
        """step() without the captured graphs (measurement passes); ordered
        after earlier graph replays by the fork from the current stream."""
        if self._events_captured:
            self._step_events()
        self.prime()
        main = torch.cuda.current_stream()
        main.wait_stream(self.s_result)
        main.wait_stream(self.s_sample)
        self._step_body(self.k)
        self.k += 1

    def store_result(self, j: int, host_ids_dev: int, host_meta_dev: int) -> None:
        """After step j: hand round j's distinct IDs (the AccessTrace row) and
        the cache counters to mapped pinned host memory (bgl_d2h_result) on a
        side stream -- no host synchronisation, off the next step's path."""
        s = self.samplers[j % self.NSMP]
        self.s_result.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.s_result):
            _lib.call("bgl_d2h_result", s.uniq.data_ptr(), s.num_uniq.data_ptr(), s.max_uniq,
                      self.counters.data_ptr(), host_ids_dev, host_meta_dev, _lib.stream_ptr(self.s_result))
            self.reported[j % self.NSMP].record(self.s_result)

    # -- results of a completed round j (host views; synchronising) ----------------
    def distinct(self, j: int) -> torch.Tensor:
        s = self.samplers[j % self.NSMP]
        return s.uniq[: int(s.num_uniq.item())]

    def rows(self, j: int) -> torch.Tensor:
        n = int(self.samplers[j % self.NSMP].num_uniq.item())
        return self.out_rows[j % self.NR][:n]

    def outcome_codes(self, j: int) -> torch.Tensor:
        n = int(self.samplers[j % self.NSMP].num_uniq.item())
        return self.out_codes[j % self.NR][:n]
