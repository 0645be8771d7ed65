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
