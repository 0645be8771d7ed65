"""The fused per-mini-batch preprocessing pipeline on one B200.

One mini-batch of BGL's data path:
    stage seeds  (device-resident proximity schedule, bgl_stage_batch)
    sample       H hops, PCG64 replay, fused dedup mark (bgl_sample_hop x H)
    dedup        sorted distinct set                    (bgl_unique_sorted)
    lookup       FIFO cache, pre-batch state            (bgl_cache_lookup)
    gather       hits from HBM ring slots, misses zero-copy from pinned host
                 (bgl_gather_rows)
    insert       insert-after-batch + row copy into the ring (bgl_cache_insert)

Software pipelining (the paper's overlap of sampling with feature retrieval,
PAPER.md:536-576): sampling is cache-independent (its rng is keyed by the
batch index, sampler.py:138), so step k runs cache+gather of batch k on one
stream while batch k+1 is sampled on another, with double-buffered sampler
and row buffers. The cache state machine still sees batches strictly in
order. Every step is captured once per buffer parity in a CUDA graph and
replayed; counts, batch index and PCG64 tables stay on the device.

Outputs of batch i (distinct IDs, rows, outcome codes, counters) equal the
reference's `simulate_epoch` trace / `simulate` report rows and
`F[trace.batches[i]]`.
"""

from __future__ import annotations

import torch

from . import _lib
from .cachesim import CacheConfig
from .features import FeatureCacheEngine
from .graph import DeviceGraph
from .sampler import BatchSampler, pcg_states, pcg_tables


class MiniBatchPipeline:
    def __init__(self, dg: DeviceGraph, fanouts, batch_size: int, order: torch.Tensor, seed: int,
                 cache_cfg: CacheConfig, features: torch.Tensor, num_batches: int | None = None,
                 sampler_ctas: int | None = None):
        if cache_cfg.num_devices != 1:
            raise ValueError("single-GPU pipeline: one cache shard (num_devices=1)")
        self.dg = dg
        self.b = int(batch_size)
        self.order = order.to(device="cuda", dtype=torch.int32).contiguous()
        total = int(self.order.numel())
        self.num_batches = int(num_batches or (total + self.b - 1) // self.b)
        if sampler_ctas is None:
            sampler_ctas = 0          # the miss gather takes only 2 warps per SM
        self.samplers = [BatchSampler(dg, fanouts, self.b, max_ctas=sampler_ctas) for _ in range(2)]
        self.max_uniq = self.samplers[0].max_uniq
        self.engine = FeatureCacheEngine(cache_cfg, features, max_batch=self.max_uniq)
        self.outs = [self.engine.out, torch.empty_like(self.engine.out)]
        self.tables = pcg_tables(pcg_states(seed, range(self.num_batches)))
        self.table_stage = [torch.empty((65, 4), dtype=torch.int64, device="cuda") for _ in range(2)]
        self.batch_counter = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.batch_index = torch.zeros(2, dtype=torch.int64, device="cuda")
        self.counters = torch.zeros(8, dtype=torch.int64, device="cuda")
        self.fed_seeds = torch.empty(self.b, dtype=torch.int32, device="cuda")
        self.fed_count = torch.zeros(1, dtype=torch.int64, device="cuda")
        # host-fed mode results: distinct IDs + {n, counters} of each batch land
        # in pinned host memory by zero-copy stores (no host sync per step)
        self.host_ids = [torch.empty(self.max_uniq, dtype=torch.int32, pin_memory=True) for _ in range(2)]
        self.host_meta = [torch.zeros(16, dtype=torch.int64, pin_memory=True) for _ in range(2)]
        self._host_ids_dev = [_lib.host_device_pointer(t) for t in self.host_ids]
        self._host_meta_dev = [_lib.host_device_pointer(t) for t in self.host_meta]
        # the cache/gather chain is the critical path (host link): its blocks are
        # dispatched ahead of the sampler's when both are pending
        self.s_stream = torch.cuda.Stream(priority=0)
        self.c_stream = torch.cuda.Stream(priority=-5)
        self.graphs: dict = {}
        self.k = 0              # batches that went through the cache
        self.primed = False     # batch k already sampled into samplers[k % 2]
        s = self.samplers[0]
        hops = 3 * s.H                                  # scan + warp + heavy per hop
        gathers = 1 if features.is_cuda else 2
        # stage, hops, dedup (mark seeds, emit, reset), lookup (fused), gather(s), insert + finalize
        self.kernels_per_step = 1 + hops + 3 + 1 + gathers + 2

    # -- building blocks ------------------------------------------------------------
    def _sample(self, slot: int, stream=None, fed: bool = False, hooks=None) -> None:
        s = self.samplers[slot]
        order = self.fed_seeds if fed else self.order
        _lib.call("bgl_stage_batch", order.data_ptr(), self.order.numel(), self.b, self.num_batches,
                  self.tables.data_ptr(), self.batch_counter.data_ptr(), s.nodes.data_ptr(), s.counts.data_ptr(),
                  self.table_stage[slot].data_ptr(), self.batch_index.data_ptr() + 8 * slot,
                  self.fed_count.data_ptr() if fed else None, _lib.stream_ptr(stream))
        s.run(self.table_stage[slot], stream=stream, hooks=hooks)

    def _cache(self, slot: int, stream=None, events=None) -> None:
        s = self.samplers[slot]
        self.engine.retrieve_device(s.uniq, s.num_uniq, s.max_uniq, 0, counters=self.counters, stream=stream,
                                    out=self.outs[slot], events=events)

    def prime(self, fed: bool = False) -> None:
        """Sample the first batch (pipeline prologue, untimed)."""
        if not self.primed:
            self._sample(self.k % 2, fed=fed)
            self.primed = True

    # -- one overlapped step: cache(k) || sample(k+1) ------------------------------
    def _overlapped(self, parity: int, fed: bool, stream=None) -> None:
        cur = torch.cuda.current_stream() if stream is None else stream
        self.s_stream.wait_stream(cur)
        self.c_stream.wait_stream(cur)
        with torch.cuda.stream(self.s_stream):
            self._sample(1 - parity, stream=self.s_stream, fed=fed)
        with torch.cuda.stream(self.c_stream):
            self._cache(parity, stream=self.c_stream)
            if fed:
                s = self.samplers[parity]
                _lib.call("bgl_d2h_result", s.uniq.data_ptr(), s.num_uniq.data_ptr(), s.max_uniq,
                          self.counters.data_ptr(), self._host_ids_dev[parity], self._host_meta_dev[parity],
                          _lib.stream_ptr(self.c_stream))
        cur.wait_stream(self.s_stream)
        cur.wait_stream(self.c_stream)

    def step_eager(self, fed: bool = False) -> None:
        self.prime(fed)
        self._overlapped(self.k % 2, fed)
        self.k += 1

    def step_serial(self, events) -> None:
        """Same work, serialised on the current stream with 6 events recorded
        around sample(k+1), dedup, lookup, gather and insert of batch k
        (stage breakdown; not used for the headline number)."""
        self.prime()
        parity = self.k % 2
        s = self.samplers[1 - parity]
        events[0].record()
        self._sample(1 - parity, hooks=lambda h: events[1].record() if h == s.H - 1 else None)
        events[2].record()
        self._cache(parity, events=events[3:6])
        self.k += 1

    def capture(self, fed: bool = False) -> None:
        """Capture the overlapped step for both buffer parities."""
        self.prime(fed)
        torch.cuda.synchronize()
        saved = self.batch_counter.clone()
        for parity in (0, 1):
            g = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cs):
                with torch.cuda.graph(g, stream=cs):
                    self._overlapped(parity, fed, stream=cs)
            torch.cuda.current_stream().wait_stream(cs)
            self.graphs[(parity, fed)] = g
        torch.cuda.synchronize()
        self.batch_counter.copy_(saved)        # capture does not execute; keep the counter exact

    def step(self, fed: bool = False) -> None:
        g = self.graphs.get((self.k % 2, fed))
        if g is None:
            self.step_eager(fed)
            return
        self.prime(fed)
        g.replay()
        self.k += 1

    def host_result(self, slot: int):
        """(distinct IDs, counters) of the last host-fed batch that used
        `slot`, read from pinned host memory (valid after a sync)."""
        n = int(self.host_meta[slot][0])
        return self.host_ids[slot][:n], self.host_meta[slot][1:9]

    # -- views of the last batch through the cache -----------------------------
    def last_slot(self) -> int:
        return (self.k - 1) % 2

    def distinct(self) -> torch.Tensor:
        return self.samplers[self.last_slot()].distinct()

    def rows(self) -> torch.Tensor:
        n = int(self.samplers[self.last_slot()].num_uniq.item())
        return self.outs[self.last_slot()][:n]

    def codes(self) -> torch.Tensor:
        n = int(self.samplers[self.last_slot()].num_uniq.item())
        return self.engine.codes[:n]

    def reset(self) -> None:
        """Cold cache, batch 0 next (graphs stay valid)."""
        torch.cuda.synchronize()
        _lib.call("bgl_cache_reset", self.engine.dev.handle, _lib.stream_ptr())
        self.counters.zero_()
        self.batch_counter.zero_()
        self.k = 0
        self.primed = False
        torch.cuda.synchronize()
