"""The fused per-mini-batch preprocessing pipeline on one B200.

One mini-batch of BGL's data path:
    stage   seeds + PCG64 table of the batch (bgl_stage_batch)
    sample  H hops, PCG64 replay, fused dedup mark (bgl_sample_hop x H)
    dedup   sorted distinct set                    (bgl_unique_sorted)
    LI      FIFO lookup vs the pre-batch state (bgl_cache_lookup) and the
            insert-after-batch of indices/rings (bgl_cache_insert_plan)
    miss    misses' rows zero-copy from pinned host memory over the host
            link (bgl_gather_rows, misses only)
    back    hits' rows from the HBM ring slots (bgl_gather_rows, hits only),
            then the survivors' rows into their new slots (bgl_cache_copy_rows)

Software pipeline (the paper overlaps sampling with feature retrieval,
PAPER.md:536-576). Step k runs five concurrent branches

    back(k)  ||  miss(k+1)  ||  LI(k+2)  ||  b(k+3)  ||  a(k+4)

(a = staging + hops 0..H-2, b = the last hop + dedup: the latency-bound
small hops of one batch fill the GPU beside the large last hop of another)

so the host link streams misses back to back while the cache bookkeeping of
the next batch, the ring-row work of the previous one and the sampling of
later ones run beside it. Dependencies all point to earlier steps: LI(k+2)
needs LI(k+1) (index state) and sample(k+2); miss(k+1) needs LI(k+1);
back(k) needs miss(k) and back(k-1); within back(k) the hits are read before
any survivor row is written (the same-batch eviction hazard). A
later LI may re-assign a slot whose row back(k) is still writing: the row is
fixed by that batch's own back() before any batch can hit the new occupant.
Sampling is cache-independent (rng keyed by the batch index,
sampler.py:138). The cache state machine therefore sees batches strictly in
order and every output equals the reference's. Buffers: samplers by batch %
5, rows / codes / src rows / insert plans by batch % 3, host-fed seeds by
batch % 2; the step is captured once per phase (k % 30) in a CUDA graph and
replayed.
"""

from __future__ import annotations

import os

import torch

from . import _lib
from .cachesim import CacheConfig
from .features import FeatureCacheEngine
from .graph import DeviceGraph
from .sampler import BatchSampler, pcg_states, pcg_tables

NS, NB = 5, 3          # sampler buffers, row/plan buffers
NF = 2                 # host-fed seed buffers
PHASES = 30            # lcm(NS, NB, NF)


def check_num_batches(num_batches, total: int, b: int) -> int:
    """Batches per epoch of a schedule of `total` seeds in batches of `b`
    (the last may be short, ordering.py:148-151). An explicit count beyond
    ceil(total / b) would stage batches past the schedule's end."""
    if b < 1:
        raise ValueError("batch_size must be >= 1")
    full = (total + b - 1) // b
    if full < 1:
        raise ValueError("empty schedule")
    nb = int(num_batches or full)
    if not 1 <= nb <= full:
        raise ValueError(f"num_batches must be in [1, {full}] for {total} seeds in batches of {b}")
    return nb


class MiniBatchPipeline:
    lookahead = 4      # batch k+4 is staged (and its first hops sampled) during step k

    def __init__(self, dg: DeviceGraph, fanouts, batch_size: int, order: torch.Tensor, seed: int,
                 cache_cfg: CacheConfig, features: torch.Tensor, num_batches: int | None = None,
                 sampler_ctas: int = 0, rng: str = "replay"):
        if cache_cfg.num_devices != 1:
            raise ValueError("single-GPU pipeline: one cache shard (num_devices=1)")
        self.dg = dg
        self.b = int(batch_size)
        self.order = order.to(device="cuda", dtype=torch.int32).contiguous()
        total = int(self.order.numel())
        self.num_batches = check_num_batches(num_batches, total, self.b)
        if not sampler_ctas:   # BGL_SAMPLER_CTAS: cap the sampler's CTAs so other branches co-run (A/B)
            sampler_ctas = int(os.environ.get("BGL_SAMPLER_CTAS", "0"))
        self.samplers = [BatchSampler(dg, fanouts, self.b, max_ctas=sampler_ctas, rng=rng, frontier_outputs=False)
                         for _ in range(NS)]
        self.max_uniq = self.samplers[0].max_uniq
        self.engine = FeatureCacheEngine(cache_cfg, features, max_batch=self.max_uniq)
        self.outs = [self.engine.out] + [torch.empty_like(self.engine.out) for _ in range(NB - 1)]
        self.codes_buf = [torch.empty(self.max_uniq, dtype=torch.uint8, device="cuda") for _ in range(NB)]
        self.src_row = [torch.empty(self.max_uniq, dtype=torch.int64, device="cuda") for _ in range(NB)]
        self.plans = [self.engine.plan_buffers() for _ in range(NB)]
        # compacted device-miss positions of each batch (written by the lookup)
        self.miss_pos = [torch.empty(self.max_uniq, dtype=torch.int32, device="cuda") for _ in range(NB)]
        self.miss_count = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(NB)]
        self.compact_misses = True
        # HBM-resident features: no host link to keep busy, so the misses are
        # gathered in the back stage's pass over the batch (one kernel, rows
        # from the ring or the table) instead of a miss stage of their own
        self.fused_hbm_gather = bool(getattr(features, "is_cuda", False)) and \
            os.environ.get("BGL_HBM_FUSED", "1") != "0"
        self.tables = pcg_tables(pcg_states(seed, range(self.num_batches)))
        self.table_stage = [torch.empty((_lib.PCG_TABLE_ROWS, 4), dtype=torch.int64, device="cuda") for _ in range(NS)]
        self.batch_counter = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.batch_index = torch.zeros(NS, dtype=torch.int64, device="cuda")
        self.counters = torch.zeros(8, dtype=torch.int64, device="cuda")
        # host-fed seeds: NF device buffers [count (int64) | seeds (int32)], each
        # filled by ONE H2D copy from a pinned staging buffer on a side stream,
        # so the copy for batch i overlaps the step in flight (feed())
        self.fed_dev = [torch.zeros(2 + self.b, dtype=torch.int32, device="cuda") for _ in range(NF)]
        self.fed_host = [torch.zeros(2 + self.b, dtype=torch.int32, pin_memory=True) for _ in range(NF)]
        self.copy_stream = torch.cuda.Stream()
        self.fed_ready = [torch.cuda.Event() for _ in range(NF)]   # H2D copy of the buffer done
        self.fed_free = [torch.cuda.Event() for _ in range(NF)]    # its batch has been staged
        # host-fed results: distinct IDs + {n, counters} of each batch stored
        # into pinned host memory by zero-copy writes (no host sync per step)
        self.host_ids = [torch.empty(self.max_uniq, dtype=torch.int32, pin_memory=True) for _ in range(NB)]
        self.host_meta = [torch.zeros(16, dtype=torch.int64, pin_memory=True) for _ in range(NB)]
        self._host_ids_dev = [_lib.host_device_pointer(t) for t in self.host_ids]
        self._host_meta_dev = [_lib.host_device_pointer(t) for t in self.host_meta]
        # back, miss, LI, sample b, sample a; the sampling branches run at high
        # stream priority: they are the critical path when the features are in
        # HBM (3757 -> 3912 b/s); no effect when the host link bounds the step
        prio = os.environ.get("BGL_STREAM_PRIO", "ab")
        self.streams = [torch.cuda.Stream(priority=-1 if (name in prio) else 0)
                        for name in ("k", "m", "l", "b", "a")]
        self.graphs: dict = {}
        self.k = 0                # batches completed (rows ready)
        self.primed = False
        s = self.samplers[0]
        # stage + H x (sample, heavy; counter RNG: one kernel per hop) + dedup (mark seeds, emit, reset)
        # + lookup + insert(2) + miss gather + hit gather + row copy (= the ncu launch list of a step);
        # host-fed: + d2h_result
        per_hop = 1 if rng == "counter" else 2
        self.kernels_per_step = 1 + per_hop * s.H + 3 + 1 + 2 + (0 if self.fused_hbm_gather else 1) + 1 + 1

    # -- stages ------------------------------------------------------------------
    def _sample(self, batch: int, stream=None, fed: bool = False, hooks=None, part: str = "all") -> None:
        """part "a": stage the batch + hops 0..H-2; "b": the last hop + dedup;
        "all": both. The pipeline runs a(k+4) beside b(k+3): the small first
        hops of one batch fill the GPU beside the big last hop of another."""
        slot = batch % NS
        s = self.samplers[slot]
        if part in ("a", "all"):
            fbuf = self.fed_dev[batch % NF].data_ptr()
            order = fbuf + 8 if fed else self.order.data_ptr()
            _lib.call("bgl_stage_batch", order, self.order.numel(), self.b, self.num_batches,
                      self.tables.data_ptr(), self.batch_counter.data_ptr(), s.nodes.data_ptr(), s.counts.data_ptr(),
                      self.table_stage[slot].data_ptr(), self.batch_index.data_ptr() + 8 * slot,
                      fbuf if fed else None, 1, 0, _lib.stream_ptr(stream))
        if part == "all":
            s.run(self.table_stage[slot], stream=stream, hooks=hooks)
        elif part == "a":
            s.run(self.table_stage[slot], stream=stream, hooks=hooks, hops=range(0, s.H - 1), dedup=False)
        else:
            s.run(self.table_stage[slot], stream=stream, hooks=hooks, hops=range(s.H - 1, s.H))

    def _li(self, batch: int, stream=None) -> None:
        s = self.samplers[batch % NS]
        j = batch % NB
        plan, pcount = self.plans[j]
        self.engine.lookup_insert(s.uniq, s.num_uniq, s.max_uniq, 0, self.codes_buf[j], self.src_row[j], plan,
                                  pcount, self.counters, stream=stream, miss_pos=self.miss_pos[j],
                                  miss_count=self.miss_count[j])

    def _miss(self, batch: int, stream=None) -> None:
        if self.fused_hbm_gather:
            return
        s = self.samplers[batch % NS]
        j = batch % NB
        if self.compact_misses:
            self.engine.miss_gather(s.uniq, s.num_uniq, s.max_uniq, self.outs[j], self.src_row[j], stream=stream,
                                    miss_pos=self.miss_pos[j], miss_count=self.miss_count[j])
        else:   # mode-2 pass over the whole batch (kept for comparison)
            self.engine.miss_gather(s.uniq, s.num_uniq, s.max_uniq, self.outs[j], self.src_row[j], stream=stream)

    def _back(self, batch: int, stream=None, fed: bool = False, events=None) -> None:
        s = self.samplers[batch % NS]
        j = batch % NB
        plan, pcount = self.plans[j]
        self.engine.back(s.uniq, s.num_uniq, s.max_uniq, self.outs[j], self.src_row[j], plan, pcount,
                         stream=stream, events=events, with_misses=self.fused_hbm_gather)
        if fed:
            _lib.call("bgl_d2h_result", s.uniq.data_ptr(), s.num_uniq.data_ptr(), s.max_uniq,
                      self.counters.data_ptr(), self._host_ids_dev[j], self._host_meta_dev[j],
                      _lib.stream_ptr(stream))

    def feed(self, batch: int, seeds) -> int:
        """Host-fed mode: queue batch `batch`'s seeds (host int sequence or
        tensor). They are staged in pinned memory and copied H2D (count +
        seeds, one copy) on a side stream, overlapping the step in flight; the
        step that samples `batch` waits for the copy. Returns the H2D bytes."""
        j = batch % NF
        seeds = torch.as_tensor(seeds)
        n = int(seeds.numel())
        if n == 0:
            raise ValueError("seeds must be nonempty")
        if n > self.b:
            raise ValueError("batch larger than the pipeline was sized for")
        self.fed_ready[j].synchronize()          # staging j's previous copy has finished
        h = self.fed_host[j]
        h[:2].view(torch.int64).fill_(n)
        h[2:2 + n].copy_(seeds.to(torch.int32))
        with torch.cuda.stream(self.copy_stream):
            self.copy_stream.wait_event(self.fed_free[j])   # its previous batch was staged
            self.fed_dev[j][:2 + n].copy_(h[:2 + n], non_blocking=True)
            self.fed_ready[j].record(self.copy_stream)
        return (2 + n) * 4

    def _fed_sample_guard(self, batch: int, before: bool) -> None:
        j = batch % NF
        if before:
            torch.cuda.current_stream().wait_event(self.fed_ready[j])
        else:
            self.fed_free[j].record(torch.cuda.current_stream())

    def prime(self, fed: bool = False, feed=None) -> None:
        """Prologue (untimed): sample k..k+2, a(k+3), LI(k), miss(k), LI(k+1).
        In host-fed mode `feed(i)` must queue batch i's seeds (self.feed)."""
        if self.primed:
            return
        for i in range(self.k, self.k + self.lookahead):
            if fed and feed is not None:
                feed(i)
            if fed:
                self._fed_sample_guard(i, True)
            self._sample(i, fed=fed, part="all" if i < self.k + self.lookahead - 1 else "a")
            if fed:
                self._fed_sample_guard(i, False)
        self._li(self.k)
        self._miss(self.k)
        self._li(self.k + 1)
        self.primed = True

    # -- one overlapped step: back(k) || miss(k+1) || LI(k+2) || b(k+3) || a(k+4) ----
    def _overlapped(self, k: int, fed: bool, stream=None) -> None:
        cur = torch.cuda.current_stream() if stream is None else stream
        sb, sm, sl, ss, sa = self.streams
        for s in self.streams:
            s.wait_stream(cur)
        with torch.cuda.stream(sm):
            self._miss(k + 1, stream=sm)
        with torch.cuda.stream(sl):
            self._li(k + 2, stream=sl)
        with torch.cuda.stream(sb):
            self._back(k, stream=sb, fed=fed)
        with torch.cuda.stream(ss):
            self._sample(k + 3, stream=ss, fed=fed, part="b")
        with torch.cuda.stream(sa):
            self._sample(k + 4, stream=sa, fed=fed, part="a")
        for s in self.streams:
            cur.wait_stream(s)

    def step_eager(self, fed: bool = False) -> None:
        self.prime(fed)
        if fed:
            self._fed_sample_guard(self.k + self.lookahead, True)
        self._overlapped(self.k, fed)
        if fed:
            self._fed_sample_guard(self.k + self.lookahead, False)
        self.k += 1

    def step_serial(self, events) -> None:
        """The same work serialised on the current stream, 7 events:
        [sample | dedup | LI | miss gather | hit gather | row copy] of one
        step (stage breakdown only)."""
        self.prime()
        k = self.k
        s = self.samplers[(k + 3) % NS]
        events[0].record()
        self._sample(k + 4, part="a")     # hops 0..H-2 of batch k+4 + the last hop of k+3 = one batch's hops
        self._sample(k + 3, part="b", hooks=lambda h: events[1].record() if h == s.H - 1 else None)
        events[2].record()
        self._li(k + 2)
        events[3].record()
        self._miss(k + 1)
        events[4].record()
        self._back(k, events=events[5:6])
        events[6].record()
        self.k += 1

    def capture(self, fed: bool = False) -> None:
        """Capture the overlapped step for every phase k % PHASES."""
        self.prime(fed)
        torch.cuda.synchronize()
        saved = self.batch_counter.clone()
        for phase in range(PHASES):
            g = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cs):
                with torch.cuda.graph(g, stream=cs):
                    self._overlapped(phase, fed, stream=cs)
            torch.cuda.current_stream().wait_stream(cs)
            self.graphs[(phase, fed)] = g
        torch.cuda.synchronize()
        self.batch_counter.copy_(saved)        # capture does not execute; keep the counter exact

    def step(self, fed: bool = False) -> None:
        g = self.graphs.get((self.k % PHASES, fed))
        if g is None or not self.primed:
            self.step_eager(fed)
            return
        if fed:
            self._fed_sample_guard(self.k + self.lookahead, True)
        g.replay()
        if fed:
            self._fed_sample_guard(self.k + self.lookahead, False)
        self.k += 1

    # -- results of the last completed batch (k - 1) -----------------------------
    def last_batch(self) -> int:
        return self.k - 1

    def last_slot(self) -> int:
        return (self.k - 1) % NB

    def distinct(self) -> torch.Tensor:
        return self.samplers[(self.k - 1) % NS].distinct()

    def rows(self) -> torch.Tensor:
        n = int(self.samplers[(self.k - 1) % NS].num_uniq.item())
        return self.outs[(self.k - 1) % NB][:n]

    def codes(self) -> torch.Tensor:
        n = int(self.samplers[(self.k - 1) % NS].num_uniq.item())
        return self.codes_buf[(self.k - 1) % NB][:n]

    def host_result(self, slot: int):
        """(distinct IDs, counters) stored into pinned host memory by the last
        host-fed batch that used row slot `slot` (valid after a sync)."""
        n = int(self.host_meta[slot][0])
        return self.host_ids[slot][:n], self.host_meta[slot][1:9]

    def reset(self) -> None:
        """Cold cache, batch 0 next (graphs stay valid)."""
        torch.cuda.synchronize()
        _lib.call("bgl_cache_reset", self.engine.dev.handle, _lib.stream_ptr())
        for smp in self.samplers:          # the batch staged by the last a() never ran its dedup
            smp.clear_marks()
        self.counters.zero_()
        self.batch_counter.zero_()
        self.k = 0
        self.primed = False
        torch.cuda.synchronize()
