"""Node-ID-sharded FIFO feature cache across GPUs (one process per GPU).

The reference routes every queried node to its home device `v % d`
(cachesim.py:505-506): a hit on the worker's own device is D, on another
device P (peer), and device misses are inserted into their home level after
the batch in ascending ID order (cachesim.py:527-528). The reference only
*simulates* the d devices in one loop; here the d levels are d GPUs:

  round j: rank w samples batch i = j*d + w (batch rng keyed by i, so the
           sampler needs no exchange; worker of batch i is i % d as in
           cachesim.py:495)
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

The host level of the reference is a single shared level (cachesim.py:388);
it is not sharded, so the multi-GPU engine requires host_capacity == 0 (the
single-process engine covers it exactly).

`ShardedFeatureCache` is written against two small interfaces -- `ops`
(partition / scatter) and `engine` (serve one worker's bucket) -- whose
product implementations are the CUDA kernels below; the CPU gloo tests plug
the test oracle in to check the exchange protocol without GPUs.
"""

from __future__ import annotations

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
