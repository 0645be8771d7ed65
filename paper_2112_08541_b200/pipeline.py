"""The fused per-mini-batch preprocessing pipeline on one B200.

One step = one mini-batch of BGL's data path:
    stage seeds  (device-resident proximity schedule, bgl_stage_batch)
    sample       H hops, PCG64 replay                 (bgl_sample_hop x H)
    dedup        sorted distinct set                   (bgl_unique_sorted)
    lookup       FIFO cache, pre-batch state           (bgl_cache_lookup)
    gather       hits from HBM ring slots, misses zero-copy from pinned host
                 (bgl_gather_rows)
    insert       insert-after-batch + row copy into the ring (bgl_cache_insert)

Everything is device-resident (counts, batch index, PCG64 tables), so the
whole step is captured once in a CUDA graph and replayed per batch; the
outputs of batch i (distinct IDs, feature rows, outcome codes, counters) are
exactly the reference's `simulate_epoch` trace / `simulate` report rows and
`F[trace.batches[i]]`.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .cachesim import CacheConfig
from .features import FeatureCacheEngine
from .graph import DeviceGraph
from .sampler import BatchSampler, pcg_states, pcg_tables


class MiniBatchPipeline:
    def __init__(self, dg: DeviceGraph, fanouts, batch_size: int, order: torch.Tensor, seed: int,
                 cache_cfg: CacheConfig, features: torch.Tensor, num_batches: int | None = None):
        if cache_cfg.num_devices != 1:
            raise ValueError("single-GPU pipeline: one cache shard (num_devices=1)")
        self.dg = dg
        self.b = int(batch_size)
        self.order = order.to(device="cuda", dtype=torch.int32).contiguous()
        total = int(self.order.numel())
        self.num_batches = int(num_batches or (total + self.b - 1) // self.b)
        self.sampler = BatchSampler(dg, fanouts, self.b)
        self.engine = FeatureCacheEngine(cache_cfg, features, max_batch=self.sampler.max_uniq)
        self.tables = pcg_tables(pcg_states(seed, range(self.num_batches)))
        self.table_stage = torch.empty((65, 4), dtype=torch.int64, device="cuda")
        self.batch_counter = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.batch_index = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.counters = torch.zeros(8, dtype=torch.int64, device="cuda")
        self.graph: torch.cuda.CUDAGraph | None = None
        self.kernels_per_step = self._count_kernels()

    def _count_kernels(self) -> int:
        hops = sum(3 if f > 32 else 2 for f in self.sampler.eff)   # scan + warp (+ block)
        return 1 + hops + 3 + 4 + 1 + 2                              # stage, hops, dedup, lookup, gather, insert

    # -- one step, eager -------------------------------------------------------
    def step_eager(self, stream=None, events=None) -> None:
        """events (optional, eager only): 6 CUDA events recorded after staging,
        sampling, dedup, lookup, gather and insert -> per-stage times."""
        s = self.sampler
        _lib.call("bgl_stage_batch", self.order.data_ptr(), self.order.numel(), self.b, self.num_batches,
                  self.tables.data_ptr(), self.batch_counter.data_ptr(), s.nodes.data_ptr(), s.counts.data_ptr(),
                  self.table_stage.data_ptr(), self.batch_index.data_ptr(), _lib.stream_ptr(stream))
        if events is None:
            s.run(self.table_stage, stream=stream)
            self.engine.retrieve_device(s.uniq, s.num_uniq, s.max_uniq, 0, counters=self.counters, stream=stream)
            return
        events[0].record()
        s.run(self.table_stage, stream=stream, hooks=lambda h: events[1].record() if h == s.H - 1 else None)
        events[2].record()
        self.engine.retrieve_device(s.uniq, s.num_uniq, s.max_uniq, 0, counters=self.counters, stream=stream,
                                    events=events[3:6])

    # -- CUDA graph ------------------------------------------------------------
    def capture(self) -> None:
        """Capture one step; replays advance the device batch counter."""
        saved = self.batch_counter.clone()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                self.step_eager(stream=side)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.batch_counter.copy_(saved)        # capture does not execute; keep the counter exact
        self.graph = g

    def step(self) -> None:
        if self.graph is None:
            self.step_eager()
        else:
            self.graph.replay()

    # -- views -----------------------------------------------------------------
    def rows(self) -> torch.Tensor:
        return self.engine.out[: int(self.sampler.num_uniq.item())]

    def distinct(self) -> torch.Tensor:
        return self.sampler.distinct()

    def reset_cache(self) -> None:
        _lib.call("bgl_cache_reset", self.engine.dev.handle, _lib.stream_ptr())
        self.counters.zero_()
        self.batch_counter.zero_()
