#!/usr/bin/env python
"""Benchmark of the B200-native BGL per-mini-batch preprocessing path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl bgl|reference]
                    [--config c2|c1] [--features host|hbm]

One step = one mini-batch: 3-hop sampling (PCG64 replay) + dedup + FIFO
cache lookup + feature gather (hits from HBM ring slots, misses zero-copy
from pinned host memory) + insert-after-batch, on the ogbn-products-shaped
synthetic graph (BASELINE.json configs[1]). Prints ONE JSON line (rank 0).

`--impl reference` times the reference algorithm on the host CPU (the numpy
oracle port of gnnio's sampler / FIFO cache + a numpy gather), with all host
cores used for the sampler (batches are independent).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c2": dict(workload="ogbn-products-shaped synthetic power-law graph (2.4M nodes, ~62M undirected edges), "
                        "100-d fp32 features in pinned host memory, GraphSAGE fanout [15,10,5], batch 1024, "
                        "FIFO cache 10% of nodes in HBM, proximity (BFS, S=4) ordering",
               n=2_400_000, avg_degree=51, dim=100, labels=47, train=0.08, fanouts=(15, 10, 5), b=1024,
               cache_frac=0.10, S=4),
    "c3": dict(workload="ogbn-papers100M-shaped synthetic power-law graph (111M nodes, ~1.55B undirected edges), "
                        "128-d fp32 features (56.9 GB) in pinned host memory, fanout [15,10,5], batch 1024, "
                        "FIFO cache 10% of nodes (11.1M rows) in HBM, proximity (BFS, S=4) ordering; 1 GPU",
               n=111_059_956, avg_degree=29, dim=128, labels=172, train=0.0108, fanouts=(15, 10, 5), b=1024,
               cache_frac=0.10, S=4),
    "c5": dict(workload="1B-edge power-law graph (64M nodes, ~1B undirected edges, ~2B CSR entries), 128-d fp32 "
                        "features (32.8 GB) in pinned host memory, fanout [15,10,5], batch 1024, FIFO cache 10% of "
                        "nodes in HBM, proximity (BFS, S=4) ordering; 1 GPU",
               n=64_000_000, avg_degree=31, dim=128, labels=64, train=0.01, fanouts=(15, 10, 5), b=1024,
               cache_frac=0.10, S=4),
    "c1": dict(workload="synthetic power-law graph 100K nodes / 1M edges, 128-d fp32 features in pinned host "
                        "memory, fanout [10,5], batch 1024, FIFO cache 10% of nodes, BFS ordering",
               n=100_000, avg_degree=20, dim=128, labels=64, train=0.10, fanouts=(10, 5), b=1024,
               cache_frac=0.10, S=4),
}
METRIC = "mini-batches/sec (sample+cache+gather)"


def workload_text(cfg, features, order="proximity"):
    """The config's workload line, with the feature store's location and the
    batch ordering as run."""
    w = cfg["workload"]
    if features == "hbm":
        w = w.replace("in pinned host memory", "resident in HBM (misses gathered from HBM)")
    if order == "random":
        w = w.replace("proximity (BFS, S=4) ordering", "random-shuffle ordering (gnnio random_shuffle_schedule)")
    return w
UNIT = "mini-batches/s"
GRAPH_SEED, RUN_SEED = 1, 1


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


class L2Flush:
    """L2 flush between timed steps (outside the events): write a buffer
    larger than the 126 MB L2, then read another one, so the step starts with
    a cold AND clean L2 (the write alone leaves ~126 MB of dirty lines whose
    write-back would be charged to the step's first kernels)."""

    def __init__(self, nbytes: int = 256 << 20):
        import torch
        self.w = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        self.r = torch.ones(nbytes // 4, dtype=torch.int32, device="cuda")

    def __call__(self):
        import torch
        self.w.zero_()
        self.r.sum(dtype=torch.int64)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
            time.sleep(0.2)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                p = [x.strip() for x in line.split(",")]
                if len(p) >= 7 and p[0].isdigit():
                    rows.append(p)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [int(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k].lower() == "active"})
        busy = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": int(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


# ----------------------------------------------------------------------------- inputs

def make_graph(cfg, kind: str):
    """kind "exact": gnnio.graph.generate_power_law(n, avg_degree, seed=1,
    train, labels) itself, rebuilt bit-identically by the native generator
    (tests/golden/graphgen.npz); "continuum": the GPU continuum-limit model of
    the same generator (papers100M scale, where the sequential process alone
    would take minutes)."""
    from paper_2112_08541_b200.graph import generate_power_law_device, generate_power_law_exact_device
    gen = generate_power_law_exact_device if kind == "exact" else generate_power_law_device
    return gen(cfg["n"], cfg["avg_degree"], seed=GRAPH_SEED, train_fraction=cfg["train"], num_labels=cfg["labels"])


def graph_data(cfg, kind: str) -> str:
    if kind == "exact":
        return (f"synthetic: gnnio.graph.generate_power_law({cfg['n']}, {cfg['avg_degree']}, seed={GRAPH_SEED}, "
                f"train_fraction={cfg['train']}, num_labels={cfg['labels']}) rebuilt bit-exactly by the native "
                f"generator; hashed fp32 features")
    return "synthetic (GPU continuum-limit power-law generator, seed 1; hashed fp32 features)"


def build_inputs(cfg, features_where: str, graph_kind: str = "exact", shared=None, order_kind: str = "proximity"):
    """shared = (local_rank, local_world, barrier): host features in ONE
    /dev/shm store registered by every GPU process of the box."""
    import torch
    from paper_2112_08541_b200.features import shared_synthetic_features, synthetic_features
    from paper_2112_08541_b200.ordering import proximity_schedule_device
    t0 = time.time()
    dg = make_graph(cfg, graph_kind)
    torch.cuda.synchronize()
    t1 = time.time()
    if shared is not None and features_where == "host":
        lr, lw, barrier = shared
        feats, store_plan = shared_synthetic_features(cfg["n"], cfg["dim"], GRAPH_SEED,
                                                      f"bgl_features_{os.environ.get('MASTER_PORT', '0')}", lr, lw,
                                                      barrier)
    else:
        store_plan = None
        feats = synthetic_features(cfg["n"], cfg["dim"], seed=GRAPH_SEED,
                                   device_resident=(features_where == "hbm"))
    torch.cuda.synchronize()
    t2 = time.time()
    if order_kind == "random":      # gnnio ordering.random_shuffle_schedule(g, b, seed): one permutation
        from paper_2112_08541_b200.ordering import _train_ids
        perm = np.random.default_rng(RUN_SEED).permutation(_train_ids(dg))
        order = torch.from_numpy(perm.astype(np.int32)).cuda()
    else:
        order, _ = proximity_schedule_device(dg, cfg["S"], cfg["b"], seed=RUN_SEED)
    torch.cuda.synchronize()
    t3 = time.time()
    setup = {"graph_gen_s": round(t1 - t0, 3), "features_gen_s": round(t2 - t1, 3),
             "ordering_epoch_s": round(t3 - t2, 3)}
    if store_plan is not None:
        setup["feature_store"] = store_plan
    return dg, feats, order, setup


def host_link_peak_gbs():
    import torch
    nbytes = 256 << 20
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(8):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        dst.copy_(src, non_blocking=True)
        e.record()
        e.synchronize()
        best = max(best, nbytes / (s.elapsed_time(e) * 1e-3) / 1e9)
    return best


def host_link_zero_copy_peak_gbs(feats, rb):
    """Sequential zero-copy read rate of the pinned feature store (the first
    256 MB of rows, every row in order, through the miss-gather kernel with
    148 CTAs): the link's rate for SM-issued reads of contiguous memory."""
    import torch
    from paper_2112_08541_b200 import _lib
    from paper_2112_08541_b200.features import table_pointer
    m = min(feats.shape[0], (256 << 20) // rb)
    idx = torch.arange(m, dtype=torch.int32, device="cuda")
    cnt = torch.tensor([m], dtype=torch.int64, device="cuda")
    out = torch.empty((m, rb), dtype=torch.uint8, device="cuda")
    tab = table_pointer(feats)
    best = 0.0
    for it in range(6):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        _lib.call("bgl_gather_list", idx.data_ptr(), cnt.data_ptr(), m, idx.data_ptr(), tab, rb, out.data_ptr(),
                  None, None, 4, 148, _lib.stream_ptr())
        e.record()
        e.synchronize()
        if it:
            best = max(best, m * rb / (s.elapsed_time(e) * 1e-3) / 1e9)
    return best


# ----------------------------------------------------------------------------- CPU reference

def import_gnnio():
    """The reference package itself: `baseline/_ref` (pip-installed from
    /root/reference, travels to the GPU box with the snapshot), else the
    read-only tree of the build container; None when neither exists (the
    numpy oracle port stands in)."""
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "gnnio")):
            if p not in sys.path:
                sys.path.insert(0, p)
            import gnnio  # noqa: F401
            from gnnio import cachesim, graph, ordering, sampler
            return {"graph": graph, "sampler": sampler, "cachesim": cachesim, "ordering": ordering, "path": p}
    return None


def bench_config(cfg, args, world, csr_entries, max_degree, nb_total):
    """The `config` object of the JSON line -- built the same way by every arm
    (GPU single, GPU sharded, CPU reference) so the driver can compare them."""
    return {"workload": workload_text(cfg, args.features, args.order), "graph": args.graph,
            "num_nodes": cfg["n"], "csr_entries": int(csr_entries), "max_degree": int(max_degree),
            "feature_dim": cfg["dim"], "fanouts": list(cfg["fanouts"]), "batch": cfg["b"],
            "cache_rows_per_gpu": int(cfg["cache_frac"] * cfg["n"]) // world, "features": args.features,
            "sampler_rng": args.rng, "ordering": args.order,
            "parallelism": "single" if world == 1 else f"dp{world}: batch i on GPU i % {world}, node-ID-sharded "
                                                       f"FIFO cache (home of v = v % {world})",
            "l2": "flushed between timed steps (256 MB write, then a 256 MB read that writes the dirty lines back; "
                  "outside the events)",
            "batches_per_epoch": int(nb_total)}


_REF = {}


def _ref_sample(i):
    """One mini-batch's sampling by the reference: gnnio sample_batch keyed
    like simulate_epoch (batch_seed = batch index, sampler.py:138)."""
    r = _REF
    nb = len(r["batches"])
    if r["gnnio"] is not None:
        sp = r["gnnio"]["sampler"]
        return sp.sample_batch(r["g"], r["batches"][i % nb], r["scfg"], batch_seed=i % nb)[1]
    from oracle import sampler_oracle as so
    return so.sample_batch(r["off"], r["col"], r["batches"][i % nb], r["fanouts"], RUN_SEED, i % nb)[2]


class RefPath:
    """The reference's per-mini-batch path on the host CPU, on the same inputs
    as the GPU arm: graph = gnnio.graph.generate_power_law's (built by the C
    restatement oracle/powerlaw_ref.c, bit-identical, seconds instead of ~10
    minutes), features = the same hashed fp32 table, schedule = gnnio's own
    proximity_schedule / random_shuffle_schedule. One mini-batch =
    gnnio sample_batch (sampler.py:97-116) -> gnnio simulate(FIFO) on the
    persistent state (cachesim.py:275-363) -> numpy gather F[distinct]."""

    def __init__(self, cfg, args, arrays=None, order=None, feats=None, world: int = 1):
        from oracle import features_oracle as fo
        from oracle import graph_oracle as go
        self.ref = import_gnnio()
        self.cfg = cfg
        n, dim = cfg["n"], cfg["dim"]
        t0 = time.time()
        if arrays is None:
            if args.graph != "exact":
                raise SystemExit("--impl reference builds the reference's own graph (--graph exact)")
            off, col, train, labels = go.generate_power_law_c(n, cfg["avg_degree"], GRAPH_SEED, cfg["train"],
                                                              cfg["labels"])
        else:
            off, col, train, labels = arrays
        t1 = time.time()
        self.off, self.col, self.train = off, col, train
        self.max_degree = int(np.diff(off).max()) if n else 0
        if feats is None:
            feats = np.empty((n, dim), dtype=np.float32)
            step = 1 << 18
            for lo in range(0, n, step):
                hi = min(n, lo + step)
                feats[lo:hi] = fo.synthetic_features(np.arange(lo, hi), dim, seed=GRAPH_SEED)
        self.feats = feats
        self.world = world
        cap = int(cfg["cache_frac"] * n) // world     # per device, as the GPU arms shard it
        t2 = time.time()
        b = cfg["b"]
        if self.ref is not None:
            G = self.ref["graph"].Graph
            self.g = G(num_nodes=n, num_edges=int(col.size), row_offsets=off, col_indices=col, labels=labels,
                       train_mask=train, feature_dim=dim)
            od = self.ref["ordering"]
            if order is not None:
                sched = [np.asarray(order[i:i + b], dtype=np.int64) for i in range(0, len(order), b)]
            elif args.order == "random":
                sched = od.random_shuffle_schedule(self.g, b, seed=RUN_SEED).batches
            else:
                sched = od.proximity_schedule(self.g, cfg["S"], b, seed=RUN_SEED).batches
            self.scfg = self.ref["sampler"].SamplingConfig(fanouts=tuple(cfg["fanouts"]), batch_size=b, seed=RUN_SEED)
            cs = self.ref["cachesim"]
            self.ccfg = cs.CacheConfig(device_capacity=cap, num_devices=world, policy="fifo",
                                       feature_bytes_per_node=dim * 4)
            self.state = cs.cold_state(self.ccfg)
            self.kind = "reference"
        else:
            from oracle import cache_oracle as co
            from oracle import ordering_oracle as oo
            self.g, self.scfg = None, None
            if order is not None:
                sched = [np.asarray(order[i:i + b], dtype=np.int64) for i in range(0, len(order), b)]
            elif args.order == "random":
                perm = np.random.default_rng(RUN_SEED).permutation(np.flatnonzero(train))
                sched = [perm[i:i + b] for i in range(0, perm.size, b)]
            else:
                sched = oo.proximity_schedule(off, col, train, cfg["S"], b, RUN_SEED)
            self.fifo = co.FifoEngine(cap, 0, world)
            self.kind = "port"
        self.batches = sched
        _REF.update(gnnio=self.ref, g=self.g, scfg=self.scfg, batches=sched, off=off, col=col,
                    fanouts=tuple(cfg["fanouts"]))
        self.setup = {"graph_s": round(t1 - t0, 2), "features_s": round(t2 - t1, 2),
                      "schedule_s": round(time.time() - t2, 2)}

    def what(self) -> str:
        if self.kind == "reference":
            return f"gnnio (the reference package, {self.ref['path']})"
        return "the numpy oracle port of gnnio (reference package not found)"

    def cache_and_gather(self, i: int, distinct) -> int:
        """FIFO simulate of batch i on the persistent state (worker i % d,
        cachesim.py:309) + F[distinct]."""
        w = i % self.world
        if self.kind == "reference":
            sp, cs = self.ref["sampler"], self.ref["cachesim"]
            cs.simulate(sp.AccessTrace(batches=[distinct]), self.ccfg, batch_devices=[w], state=self.state)
        else:
            self.fifo.run([distinct], [w])
        rows = self.feats[distinct]
        return int(rows.nbytes)

    def run(self, idx, procs: int):
        """Batches `idx` in order: sampling in a pool of `procs` processes
        (batches are independent), the cache state machine and
        the gather in this process in batch order as the samples arrive."""
        import multiprocessing as mp
        t0 = time.time()
        fb, ts = 0, 0.0
        if procs > 1:
            with mp.get_context("fork").Pool(procs) as pool:
                for i, d in zip(idx, pool.imap(_ref_sample, idx, chunksize=1)):
                    t = time.time()
                    fb += self.cache_and_gather(i, d)
                    ts += time.time() - t
        else:
            for i in idx:
                d = _ref_sample(i)
                t = time.time()
                fb += self.cache_and_gather(i, d)
                ts += time.time() - t
        return {"batches": len(idx), "seconds": time.time() - t0, "cache_gather_s": ts, "feature_bytes": fb}


def host_procs(per_proc_gb: float) -> int:
    """Worker processes for the reference sampler: every core this process may
    run on, capped so the pool fits in the memory available."""
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    avail = None
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                avail = int(line.split()[1]) / 1e6
    except OSError:
        pass
    if avail:
        cores = max(1, min(cores, int(avail * 0.7 / per_proc_gb)))
    return cores


# ----------------------------------------------------------------------------- arms

def dropin_e2e(args, cfg, dg, feats, order_host, max_uniq):
    """The same window through the gnnio-signature drop-in functions, as a
    gnnio caller switching packages would run it (host-synchronous API, wall
    clock): sampler.simulate_epoch over the schedule's first W+K batches
    (sampler.py:119-167; batch rng keyed by the batch index), then per batch
    FeatureCacheEngine.retrieve (lookup + gather + insert, the rows F[batch]
    on the device; its state is the CacheEngineState that
    cachesim.simulate(trace, cfg, state=engine.state) drives), and separately
    cachesim.simulate over the same trace (cachesim.py:275-363, the counters
    only, no rows). Rows per batch are checked against the pipeline's."""
    import torch
    from paper_2112_08541_b200.cachesim import CacheConfig, simulate
    from paper_2112_08541_b200.features import FeatureCacheEngine
    from paper_2112_08541_b200.ordering import BatchSchedule
    from paper_2112_08541_b200.sampler import AccessTrace, SamplingConfig, simulate_epoch
    b, nb = cfg["b"], args.warmup + args.steps
    epoch = -(-order_host.size // b)
    # the pipeline's window wraps over the epoch (batch i % epoch): whole epochs, then the rest
    parts = [min(epoch, nb - e) for e in range(0, nb, epoch)]
    sched = BatchSchedule(batches=[order_host[i * b:(i + 1) * b].astype(np.int64) for i in range(min(nb, epoch))],
                          batch_size=b, policy="proximity")
    scfg = SamplingConfig(fanouts=tuple(cfg["fanouts"]), batch_size=b, seed=RUN_SEED, rng=args.rng)
    ccfg = CacheConfig(device_capacity=int(cfg["cache_frac"] * cfg["n"]), feature_bytes_per_node=cfg["dim"] * 4)
    eng = FeatureCacheEngine(ccfg, feats, max_uniq)
    simulate_epoch(dg, None, BatchSchedule(batches=sched.batches[:2], batch_size=b, policy="proximity"), scfg)   # warm the kernels
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rows_of = []
    for m in parts:
        tr, _ = simulate_epoch(dg, None, BatchSchedule(batches=sched.batches[:m], batch_size=b, policy="proximity"),
                               scfg)
        rows_of += tr.batches
    trace = AccessTrace(batches=rows_of)
    t1 = time.perf_counter()
    qbytes = 0
    for i, ids in enumerate(trace.batches):
        rows, codes = eng.retrieve(ids, i)
        qbytes += ids.size * 4
    codes_last = codes.cpu()                  # the step's result back on the host
    t2 = time.perf_counter()
    simulate(AccessTrace(batches=trace.batches[:2]), ccfg)     # warm: first-call allocations outside the timing
    torch.cuda.synchronize()
    t2s = time.perf_counter()
    rep = simulate(trace, ccfg)
    t3 = time.perf_counter()
    assert rep.total_queries == sum(x.size for x in trace.batches)
    return {"value": round(nb / (t2 - t0), 2), "unit": UNIT, "batches": nb,
            "api": "sampler.simulate_epoch (trace to the host) + FeatureCacheEngine.retrieve per batch (ids H2D, "
                   "rows F[batch] in HBM, codes D2H at the end); wall clock, host-synchronous gnnio-style calls",
            "simulate_epoch_ms_per_batch": round(1e3 * (t1 - t0) / nb, 3),
            "retrieve_ms_per_batch": round(1e3 * (t2 - t1) / nb, 3),
            "simulate_ms_per_batch": round(1e3 * (t3 - t2s) / nb, 3),   # cachesim.simulate over the trace (FIFO)
            "h2d_bytes_per_step": int(qbytes / nb + b * 8),
            "d2h_bytes_per_step": int(qbytes * 2 / nb + codes_last.numel() / nb)}


def cpu_baseline(cfg, args, dg, feats, order_host, nsample: int = 2):
    """The reference's CPU path (gnnio sample_batch + simulate + numpy
    gather, RefPath) timed on one core of this box on a bounded sample: the
    first `nsample` timed batches of the same schedule after the warm-up
    batches, on the same graph (copied from the device), features and cache."""
    hg = dg.to_host()
    fh = feats.cpu().numpy() if feats.is_cuda else feats.numpy()
    rp = RefPath(cfg, args, arrays=(hg.row_offsets, hg.col_indices, hg.train_mask, hg.labels), order=order_host,
                 feats=fh)
    rp.run(list(range(args.warmup)), procs=1 if args.warmup <= 1 else min(args.warmup, host_procs(2.0)))
    r = rp.run(list(range(args.warmup, args.warmup + nsample)), procs=1)
    return {"value": round(r["batches"] / r["seconds"], 4), "unit": UNIT, "cores": 1, "kind": rp.kind,
            "sample": f"batches {args.warmup}..{args.warmup + nsample - 1} of this schedule after the "
                      f"{args.warmup} warm-up batches (their cache state replayed untimed): {rp.what()} "
                      f"sample_batch + FIFO simulate + numpy F[distinct], 1 core, {r['seconds']:.1f}s "
                      f"({r['cache_gather_s']:.2f}s cache + gather)"}


def run_bgl(args, cfg):
    import torch
    import torch.distributed as dist
    from paper_2112_08541_b200.cachesim import CacheConfig
    from paper_2112_08541_b200.pipeline import MiniBatchPipeline

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    peak_first = host_link_peak_gbs()           # before the feature store is pinned
    dg, feats, order, setup = build_inputs(cfg, args.features, args.graph, order_kind=args.order)
    b = cfg["b"]
    cap = int(cfg["cache_frac"] * cfg["n"]) // world
    rb = cfg["dim"] * 4
    nb_total = (order.numel() + b - 1) // b
    pipe = MiniBatchPipeline(dg, cfg["fanouts"], b, order, RUN_SEED,
                             CacheConfig(device_capacity=cap, feature_bytes_per_node=rb), feats, rng=args.rng)
    pipe.step_eager()                       # warm the kernels before capture
    pipe.step_eager()
    torch.cuda.synchronize()
    pipe.capture()
    pipe.capture(fed=True)
    pipe.reset()
    peak_host = host_link_peak_gbs()
    flush = L2Flush()

    pipe.prime()
    for _ in range(args.warmup):
        pipe.step()
    torch.cuda.synchronize()
    c0 = pipe.counters.clone()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for k in range(args.steps):
            flush()                  # L2 flush between timed steps (outside the events)
            ev[k][0].record()
            pipe.step()                    # graph: cache+gather of batch k || sampling of batch k+1
            ev[k][1].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in ev]
    total_ms = sum(step_ms)
    c1 = pipe.counters.clone()
    d = (c1 - c0).cpu().tolist()
    queries, hits = d[0], d[1] + d[2] + d[3]
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        q = torch.tensor([queries, hits], dtype=torch.int64, device="cuda")
        dist.all_reduce(q)
        queries, hits = q.tolist()

    # stage breakdown + gather roofline (serialised steps with events, after the timed region)
    R = 10
    st_times = {k: [] for k in ("sample", "dedup", "lookup_insert", "miss_gather", "hit_gather", "row_copy")}
    g_bytes_host, g_ms, hbm_bytes, hbm_ms = [], [], [], []
    hist = []                                  # lookup counters per step: batch k+2 of step k
    for _ in range(R):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
        cb = pipe.counters.clone()
        flush()
        pipe.step_serial(evs)                  # a(k+4) + b(k+3) | LI(k+2) | miss(k+1) | back(k)
        torch.cuda.synchronize()
        hist.append((pipe.counters - cb).cpu().tolist())
        t = [evs[i].elapsed_time(evs[i + 1]) for i in range(6)]
        for k, v in zip(st_times, t):
            st_times[k].append(v)
        if len(hist) >= 2:                     # miss(k+1): H + M rows of batch k+1 (looked up last step)
            ca = hist[-2]
            g_bytes_host.append((ca[3] + ca[4]) * rb)
            g_ms.append(t[3])
        if len(hist) >= 3:                     # back(k): D + P rows of batch k (looked up two steps ago)
            ca = hist[-3]
            # fused HBM gather: back(k) reads + writes every row of batch k
            hbm_bytes.append(2 * ((ca[1] + ca[2] + ca[3] + ca[4]) if pipe.fused_hbm_gather else (ca[1] + ca[2])) * rb)
            hbm_ms.append(t[4])
    # host-link peak sampled twice (before the timed region and right after
    # the stage breakdown): the link rate of the pool's boxes drifts a few GB/s
    peak_samples = [peak_first, peak_host, host_link_peak_gbs()]
    peak_zc = host_link_zero_copy_peak_gbs(feats, rb) if args.features == "host" else 0.0
    peak_host = max(peak_samples + [peak_zc])
    gather_ms = statistics.mean(g_ms)
    host_bytes = statistics.mean(g_bytes_host)
    if args.features == "host":
        # the timed steps' own miss bytes over the timed time: the K lookups of
        # the window (batches W+2 .. W+K+1; step k gathers batch k+1's misses,
        # so the window's gathers are batches W+1 .. W+K: one batch shifted)
        miss_bytes_timed = (d[3] + d[4]) * rb
        achieved = miss_bytes_timed / (total_ms * 1e-3) / 1e9
        kernel_alone = host_bytes / (gather_ms * 1e-3) / 1e9
        roof = {"bound": "host_link", "achieved": round(achieved, 2), "peak": round(peak_host, 2), "unit": "GB/s",
                "frac": round(achieved / peak_host, 3),
                "traffic": None, "kernel": "gather_span_kernel (compacted misses: TMA spans + 16-B zero-copy host reads)",
                "achieved_method": "H+M rows of the timed steps' lookups x row bytes / the timed steps' CUDA-event "
                                   "time (the step is the miss gather, the other branches run beside it)",
                "achieved_serialised_kernel": round(kernel_alone, 2),
                "algorithmic_bytes_per_launch": int(miss_bytes_timed / max(args.steps, 1)),
                "peak_source": "max over this run of the pinned host->device cudaMemcpy (256 MB, best of 8; at "
                               "start-up, before the timed region, after the stage breakdown: "
                               f"{[round(x, 2) for x in peak_samples]}) and a sequential zero-copy read of 256 MB "
                               f"of the feature store ({round(peak_zc, 2)}); the host link is not in "
                               "MEASURED_PEAKS.json"}
    else:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
            if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
        # both gathers read HBM here: misses (front) and hits (back), 2 x rows x rb each; fused: one
        # gather_v4 pass over the whole batch in back(k), timed alone (the empty miss stage is not added)
        if pipe.fused_hbm_gather:
            alg = statistics.mean(hbm_bytes)
            t_g = statistics.mean(hbm_ms)
        else:
            alg = statistics.mean(g_bytes_host) * 2 + statistics.mean(hbm_bytes)
            t_g = gather_ms + statistics.mean(hbm_ms)
        achieved = alg / (t_g * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 3), "traffic": None,
                "kernel": ("gather_v4_kernel (every row in one pass: hits from the HBM ring, misses from the "
                           "HBM-resident table)" if pipe.fused_hbm_gather else
                           "gather_span_kernel (misses) + gather_v4_kernel (hits), one launch each"),
                "algorithmic_bytes_per_launch": int(alg)}
    prof = os.path.join(ROOT, "profiles", f"traffic_{args.config}_{args.features}.json")
    if os.path.exists(prof):
        tr = json.load(open(prof))
        if args.features == "host":
            # bytes that crossed the host link per miss-gather launch (ncu pcie__read_bytes)
            roof["traffic"] = tr["miss_gather"]["pcie_read_bytes_per_launch"]
            roof["traffic_kind"] = "pcie_read_bytes (ncu, one launch)"
            roof["traffic_launch_algorithmic_bytes"] = tr["miss_gather"].get("algorithmic_bytes_per_launch")
        elif pipe.fused_hbm_gather and "fused_gather" in tr:
            roof["traffic"] = tr["fused_gather"]["dram_bytes_per_launch"]
            roof["traffic_kind"] = "dram__bytes_read+write (ncu, one launch; writes that stay in L2 are not counted)"
        else:
            roof["traffic"] = tr["miss_gather"]["dram_bytes_per_launch"] + tr["hit_gather"]["dram_bytes_per_launch"]
            roof["traffic_kind"] = "dram__bytes_read+write (ncu, one launch of each gather; writes that stay in L2 are not counted)"
        roof["traffic_source"] = (tr["fused_gather"]["source"] if args.features != "host" and pipe.fused_hbm_gather
                                  and "fused_gather" in tr else tr.get("source"))

    # e2e through the public API with host buffers: every step copies the next
    # batch's seeds from pinned host memory and reads this batch's distinct IDs
    # (the AccessTrace row) and the cache counters back to pinned host memory.
    order_host = order.cpu().numpy().astype(np.int32)
    nbl = pipe.num_batches
    seeds_pinned = torch.from_numpy(order_host).pin_memory()
    out_ids = torch.empty(pipe.max_uniq, dtype=torch.int32).pin_memory()
    out_cnt = torch.empty(8, dtype=torch.int64).pin_memory()

    def feed(i):
        lo, hi = (i % nbl) * b, min((i % nbl + 1) * b, order_host.size)
        return pipe.feed(i, seeds_pinned[lo:hi])   # staged + one H2D copy on a side stream

    # same batch window as `value`: the same W warm-up steps (untimed, from a
    # cold cache), then the same K timed steps, each bracketed like `value`
    pipe.reset()
    pipe.prime(fed=True, feed=feed)
    feed(pipe.lookahead)                           # seeds of the batch sampled in the first step
    for k in range(args.warmup):
        pipe.step(fed=True)
        feed(k + 1 + pipe.lookahead)
    torch.cuda.synchronize()
    n_e2e = args.steps
    ce0 = pipe.counters.clone()
    eev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_e2e)]
    h2d = 0
    cur = torch.cuda.current_stream()
    for k in range(args.warmup, args.warmup + n_e2e):
        flush()
        e = eev[k - args.warmup]
        e[0].record()
        cur.wait_event(pipe.fed_ready[(k + pipe.lookahead) % len(pipe.fed_ready)])   # this step's seeds are in
        pipe.step(fed=True)                        # stores the batch's results into pinned host memory
        # the next step's seeds: copied H2D on the side stream while this step runs,
        # and inside this step's timed region (the end event waits for the copy)
        h2d += feed(k + 1 + pipe.lookahead)
        cur.wait_event(pipe.fed_ready[(k + 1 + pipe.lookahead) % len(pipe.fed_ready)])
        e[1].record()
    torch.cuda.synchronize()
    e2e_ms = [s.elapsed_time(e) for s, e in eev]
    ids_h, cnt_h = pipe.host_result(pipe.last_slot())
    assert torch.equal(ids_h, pipe.distinct().cpu()), "host-side result differs from the device batch"
    u_mean = float((pipe.counters - ce0)[0].item()) / n_e2e
    d2h = int(u_mean * 4 + 9 * 8) * n_e2e

    dropin = dropin_e2e(args, cfg, dg, feats, order_host, pipe.max_uniq)

    value = world * args.steps / (total_ms * 1e-3)
    ms_per_step = total_ms / args.steps
    feat_gbs = queries * rb / (total_ms * 1e-3) / 1e9
    out = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32 ids / u53 PCG64 keys / fp32 rows moved",
        "data": graph_data(cfg, args.graph),
        "config": bench_config(cfg, args, world, dg.num_edges, dg.max_degree, nb_total),
        "feature_gbs": round(feat_gbs, 2), "hit_pct": round(100.0 * hits / max(queries, 1), 2),
        "rows_per_batch": round(queries / max(args.steps, 1) / 1, 1),
        "stages_ms": {k: round(statistics.mean(v), 4) for k, v in st_times.items()},
        **sampler_report(dg, cfg, order, args.rng, statistics.mean(st_times["sample"]),
                         statistics.mean(st_times["dedup"])),
        "roofline": roof,
        "e2e": {"value": round(n_e2e / (sum(e2e_ms) * 1e-3) * world, 2), "unit": UNIT,
                "h2d_bytes_per_step": int(h2d / n_e2e), "d2h_bytes_per_step": int(d2h / n_e2e),
                "api": "MiniBatchPipeline host-fed steps: every step stages the next batch's seeds in pinned "
                       "memory and copies them H2D (one cudaMemcpy of count + seeds on a side stream, overlapping "
                       "the step, inside its timed region); the step's distinct IDs (the AccessTrace row) + "
                       "cache counters are stored into pinned host memory by bgl_d2h_result (zero-copy, no "
                       "per-step host sync); checked on the host"},
        "e2e_dropin": dropin,
        "gpu_launches": pipe.kernels_per_step * args.steps,
        "clocks": clk.summary(),
        "setup": dict(setup, torch_alloc_peak_gb=round(torch.cuda.max_memory_allocated() / 1e9, 2)),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, args, dg, feats, order_host)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_sharded(args, cfg):
    """N GPUs, one process each: node-ID-sharded FIFO cache (home = v % N,
    cachesim.py:319-320), rank w samples batches i = j*N + w (worker i % N,
    cachesim.py:309). Default engine: ShardedPipeline -- IDs pushed to the
    homes over peer memory by the partition kernel, codes and hit rows pushed
    back by the homes, misses fetched by each worker over its own host link,
    NCCL only as a one-int barrier, no host synchronisation per round
    (paper_2112_08541_b200/distributed.py). `--exchange nccl`: the all-to-all
    baseline (ShardedFeatureCache, host-synchronised per round).
    One step = one round = N mini-batches (one per GPU).

    Shared-GPU mode (fewer visible GPUs than ranks, e.g. the 1-GPU test box):
    ranks share devices round-robin, the process group is gloo (NCCL refuses
    two ranks on one GPU), the data-path barrier is a host barrier and steps
    run eagerly -- the same kernels and peer stores (CUDA IPC within a device),
    for correctness and launcher checks, not for speed."""
    import torch
    import torch.distributed as dist
    from paper_2112_08541_b200.distributed import GpuShardEngine, GpuShardOps, ShardedFeatureCache, ShardedPipeline
    from paper_2112_08541_b200.sampler import BatchSampler, pcg_states, pcg_tables

    if "RANK" not in os.environ:            # single process without torchrun (--sharded at N=1)
        os.environ.update(RANK="0", LOCAL_RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=os.environ.get("MASTER_PORT", "29531"))
    rank, local_rank, world = dist_env()
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    ndev = torch.cuda.device_count()
    shared_gpu = ndev < local_world
    dev_index = local_rank % ndev
    torch.cuda.set_device(dev_index)
    if shared_gpu:
        dist.init_process_group("gloo")
        if args.exchange != "push":
            raise SystemExit("--exchange nccl needs one GPU per rank")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
    cpu_coll = shared_gpu

    def allreduce(t, op=dist.ReduceOp.SUM):
        if cpu_coll:
            c = t.cpu()
            dist.all_reduce(c, op=op)
            t.copy_(c)
        else:
            dist.all_reduce(t, op=op)
        return t

    def allgather_list(vals):
        out = [None] * world
        dist.all_gather_object(out, vals)
        return out

    def host_barrier():
        torch.cuda.synchronize()
        dist.barrier()

    dg, feats, order, setup = build_inputs(cfg, args.features, args.graph, order_kind=args.order,
                                           shared=(local_rank, local_world, dist.barrier) if world > 1 else None)
    b, rb, dim = cfg["b"], cfg["dim"] * 4, cfg["dim"]
    cap = int(cfg["cache_frac"] * cfg["n"]) // world
    nb_total = (order.numel() + b - 1) // b
    flush = L2Flush()
    order_host = order.cpu().numpy().astype(np.int32)
    seeds_pinned = torch.from_numpy(order_host).pin_memory()

    if args.exchange == "push":
        pipe = ShardedPipeline(rank, world, dg, cfg["fanouts"], b, order, RUN_SEED, cap, feats, rng=args.rng,
                               barrier=host_barrier if shared_gpu else None)
        counters = pipe.counters
        launches = pipe.kernels_per_round
        graphs = "off (shared-GPU mode: host barriers)" if shared_gpu else "off"
        if not args.no_graphs and not shared_gpu:
            try:
                pipe.capture()                    # one CUDA graph per step phase, NCCL barriers inside
                graphs = "on"
            except Exception as e:                # noqa: BLE001 -- report and run the same steps eagerly
                pipe.graphs.clear()
                graphs = f"capture failed ({type(e).__name__}: {str(e)[:80]}); eager"

        def one_round(j, host_fed=False):
            pipe.step()                   # step j: rows of round j complete
    else:
        graphs = "off"
        sampler = BatchSampler(dg, cfg["fanouts"], b)
        engine = GpuShardEngine(rank, world, cap, feats, sampler.max_uniq)
        sc = ShardedFeatureCache(rank, world, engine, GpuShardOps(world, sampler.max_uniq, rb), dim)
        tables = pcg_tables(pcg_states(RUN_SEED, range(nb_total)))
        counters = engine.counters
        launches = 3 * len(cfg["fanouts"]) + 4 + 3 + 5 * world

        def one_round(j, host_fed=False):
            i = (j * world + rank) % nb_total
            lo, hi = i * b, min((i + 1) * b, order.numel())
            sampler.load_seeds(seeds_pinned[lo:hi] if host_fed else order[lo:hi])
            sampler.run(tables[i])
            u = int(sampler.num_uniq.item())
            sc.step(sampler.uniq[:u])

    for j in range(args.warmup):
        one_round(j)
    torch.cuda.synchronize()
    c0 = counters.clone()
    dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(dev_index) as clk:
        for k in range(args.steps):
            flush()
            ev[k][0].record()
            one_round(args.warmup + k)
            ev[k][1].record()
        torch.cuda.synchronize()
    dist.barrier()
    total_ms_rank = sum(s.elapsed_time(e) for s, e in ev)
    d_rank = (counters - c0).clone()
    per_rank = allgather_list([int(x) for x in d_rank.cpu().tolist()] + [total_ms_rank])
    d = allreduce(d_rank.clone())
    t = allreduce(torch.tensor([total_ms_rank], dtype=torch.float64, device="cuda"), dist.ReduceOp.MAX)
    total_ms = float(t.item())
    q, own, peer, hst = (int(x) for x in d[:4].tolist())
    roof = sharded_roofline(args, pipe if args.exchange == "push" else None, feats, rb, flush, allreduce,
                            allgather_list, shared_gpu)
    # e2e: every round the next round's seeds go H2D from pinned host (on the
    # sampling stream, ahead of the sampler) and the round's distinct IDs (the
    # AccessTrace row) + counters are stored into pinned host memory
    n_e2e = max(3, min(args.steps, 50))
    from paper_2112_08541_b200 import _lib
    if args.exchange == "push":
        maxu = pipe.maxu
    else:
        maxu = sampler.max_uniq
    host_ids = torch.empty(maxu, dtype=torch.int32).pin_memory()
    host_meta = torch.zeros(16, dtype=torch.int64).pin_memory()
    hid, hmeta = _lib.host_device_pointer(host_ids), _lib.host_device_pointer(host_meta)
    eev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_e2e)]
    h2d, d2h = 0, 0
    torch.cuda.synchronize()
    for k in range(n_e2e):
        j = args.warmup + args.steps + k
        eev[k][0].record()
        if args.exchange == "push":
            i = pipe.batch_of(j + 3)      # step j samples round j + 3: its seeds come from the host
            lo, hi = i * b, min((i + 1) * b, order.numel())
            with torch.cuda.stream(pipe.s_sample):
                pipe.order[lo:hi].copy_(seeds_pinned[lo:hi], non_blocking=True)
            one_round(j)
            s = pipe.samplers[j % pipe.NSMP]
            pipe.store_result(j, hid, hmeta)       # side stream, overlapping the next step
            if k == n_e2e - 1:                     # (back-to-back steps: every hand-off ends inside the region)
                torch.cuda.current_stream().wait_stream(pipe.s_result)
        else:
            one_round(j, host_fed=True)
            s = sampler
            _lib.call("bgl_d2h_result", s.uniq.data_ptr(), s.num_uniq.data_ptr(), s.max_uniq, counters.data_ptr(),
                      hid, hmeta, _lib.stream_ptr())
        eev[k][1].record()
        h2d += (hi - lo if args.exchange == "push" else b) * 4
    torch.cuda.synchronize()
    e2e_ms = [x.elapsed_time(y) for x, y in eev]
    u_last = int(host_meta[0])
    assert torch.equal(host_ids[:u_last], s.uniq[:u_last].cpu()), "host-side result differs from the device"
    d2h = n_e2e * (u_last * 4 + 72)
    t = allreduce(torch.tensor([sum(e2e_ms)], dtype=torch.float64, device="cuda"), dist.ReduceOp.MAX)
    ranks = []
    for r, v in enumerate(per_rank):
        rq = max(v[0], 1)
        ranks.append({"rank": r, "queries": v[0], "hit_pct": round(100.0 * (v[1] + v[2] + v[3]) / rq, 2),
                      "peer_hit_pct": round(100.0 * v[2] / rq, 2), "miss_pct": round(100.0 * v[4] / rq, 2),
                      "timed_ms": round(v[8], 3)})
    out = {
        "metric": METRIC, "value": round(world * args.steps / (total_ms * 1e-3), 2), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32 ids / u53 PCG64 keys / fp32 rows moved",
        "data": graph_data(cfg, args.graph),
        "config": bench_config(cfg, args, world, dg.num_edges, dg.max_degree, nb_total),
        "engine": {"step": f"one round = {world} mini-batches (one per GPU)", "cuda_graphs": graphs,
                   "exchange": ("IDs pushed to the homes over peer memory by the partition kernel, codes and hit "
                                "rows pushed back by the homes (CUDA IPC), misses fetched by each worker over its "
                                "own host link, NCCL one-int barriers, no host sync per round"
                                if args.exchange == "push" else "IDs and rows by NCCL all-to-all (host-synchronised)"),
                   "shared_gpu": (f"{world} ranks on {ndev} visible GPU(s): gloo + host barriers, eager steps "
                                  f"(correctness/launcher mode, not a speed number)") if shared_gpu else False},
        "feature_gbs": round(q * rb / (total_ms * 1e-3) / 1e9, 2),
        "hit_pct": round(100.0 * (own + peer + hst) / max(q, 1), 2),
        "peer_hit_pct": round(100.0 * peer / max(q, 1), 2),
        "per_rank": ranks,
        "e2e": {"value": round(world * n_e2e / (float(t.item()) * 1e-3), 2), "unit": UNIT,
                "h2d_bytes_per_step": int(h2d / n_e2e), "d2h_bytes_per_step": int(d2h / n_e2e)},
        "roofline": roof,
        "gpu_launches": launches * args.steps,
        "clocks": clk.summary(), "setup": dict(setup, torch_alloc_peak_gb=round(torch.cuda.max_memory_allocated() / 1e9, 2)),
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if args.exchange == "push":
        dist.barrier()
        pipe.close()
    dist.destroy_process_group()


def sampler_report(dg, cfg, order, rng, sample_ms, dedup_ms, n=8):
    """SURVEY §8d's separate sampler / dedup figures for the replay sampler:
    PCG64 draws per batch (= steps of the replayed stream, ALU only) and their
    rate over the bench's serialised sample stage, parents and outputs per hop,
    the algorithmic bytes sum_h [P_h*16 + S_h*4 + S_h*8], dedup keys/s. Counts
    from n batches of the bench's schedule sampled once more, outside the
    timed region."""
    if rng != "replay":
        return {}
    import torch
    from paper_2112_08541_b200.sampler import BatchSampler, pcg_states, pcg_tables
    b = cfg["b"]
    s = BatchSampler(dg, cfg["fanouts"], b)
    tables = pcg_tables(pcg_states(RUN_SEED, range(n)))
    draws, counts = [], []
    for i in range(n):
        s.load_seeds(order[i * b:(i + 1) * b])
        s.run(tables[i])
        draws.append(int(s.draw_base[-1].item()))
        counts.append(s.host_counts())
    del s
    torch.cuda.empty_cache()
    c = np.mean(np.array(counts, dtype=np.float64), axis=0)
    H = len(cfg["fanouts"])
    parents, outs = c[:H], c[1:H + 1]
    d = float(np.mean(draws))
    keys = float(c.sum())
    return {"sampler": {"draws_per_batch": round(d), "pcg64_draws_per_s": round(d / (sample_ms * 1e-3)),
                        "parents_per_hop": [round(x) for x in parents], "outputs_per_hop": [round(x) for x in outs],
                        "algorithmic_bytes_per_batch": round(float(np.sum(parents * 16 + outs * 12))),
                        "bound": "integer ALU: one 128-bit LCG step + XSL-RR per draw (no bytes per draw)",
                        "stage_ms": round(sample_ms, 4)},
            "dedup": {"keys_per_batch": round(keys), "keys_per_s": round(keys / (dedup_ms * 1e-3)),
                      "stage_ms": round(dedup_ms, 4)}}


NVLINK_PEER_GBS = 770.0     # measured peer copy per direction (B200_PROFILING.md; 900 nominal)


def sharded_roofline(args, pipe, feats, rb, flush, allreduce, allgather_list, shared_gpu, R=8):
    """Roofline of the sharded engine's dominant kernel, the worker's miss
    gather (bgl_gather_spans over this rank's own device-missed rows): R eager
    steps after the timed region, events on the miss stream around the
    gathers, rows read from the step's miss counts; max over ranks of the time.
    Also the peer (NVLink) side: the rows each home pushed into other GPUs'
    outputs (its P hits) over its B stage (events on the back stream), and the
    host-link peak measured with every rank copying at once."""
    import torch
    import torch.distributed as dist
    if pipe is None:
        return {"bound": "host_link" if args.features == "host" else "hbm", "achieved": None, "peak": None,
                "unit": "GB/s", "frac": None, "traffic": None,
                "kernel": "n/a for the NCCL all-to-all baseline (--exchange nccl)"}
    world = dist.get_world_size()
    pipe.miss_timing, pipe.back_timing = [], []
    rows, peer_rows = [], []
    for _ in range(R):
        r = (pipe.k + 1) % pipe.NR               # step k gathers the misses of round k + 1
        c0 = pipe.counters.clone()
        flush()
        pipe.step_eager()
        torch.cuda.synchronize()
        rows.append(int(pipe.own_misses(r)[1].item()))   # this rank's own misses (the worker fetches them)
        # P hits served by this home (looked up in LI(k+2)); in steady state the
        # same count its B(k) pushes to other GPUs
        peer_rows.append(int((pipe.counters - c0)[2].item()))
    ms = sum(a.elapsed_time(b) for a, b, _ in pipe.miss_timing)
    bms = sum(a.elapsed_time(b) for a, b in pipe.back_timing)
    pipe.miss_timing, pipe.back_timing = None, None
    t = allreduce(torch.tensor([ms, bms], dtype=torch.float64, device="cuda"), dist.ReduceOp.MAX)
    tot = allreduce(torch.tensor([float(sum(rows)), float(sum(peer_rows))], dtype=torch.float64, device="cuda"))
    tmax, bmax = float(t[0].item()), float(t[1].item())
    per_rank_bytes = float(tot[0].item()) / world * rb
    peer_bytes = float(tot[1].item()) / world * rb
    nvl = {"peer_push_bytes_per_round": int(peer_bytes / R), "b_stage_ms_per_round": round(bmax / R, 4),
           "achieved": round(peer_bytes / (bmax * 1e-3) / 1e9, 2) if bmax > 0 else None, "unit": "GB/s",
           "peak": NVLINK_PEER_GBS,
           "peak_source": "measured peer copy per direction, /opt/skills/guides/B200_PROFILING.md (900 nominal)",
           "kernel": "gather_v4_kernel in home-push mode (bgl_gather_rows_push: ring hits stored into the worker "
                     "GPU's output over peer memory) + the ring survivor copy, per home over its B stage"}
    if nvl["achieved"] is not None:
        nvl["frac"] = round(nvl["achieved"] / NVLINK_PEER_GBS, 3)
    if shared_gpu:
        nvl["note"] = "shared-GPU mode: the 'peer' stores stay inside one device (no NVLink crossed)"
    if args.features == "host":
        dist.barrier()
        alone = host_link_peak_gbs()
        dist.barrier()
        together = host_link_peak_gbs()          # every rank copying at once
        peaks = allgather_list([alone, together])
        try:
            zc = host_link_zero_copy_peak_gbs(feats, rb)
        except Exception:  # noqa: BLE001 -- a shared store without .shape: memcpy samples only
            zc = 0.0
        # the link rate a rank gets while all ranks copy (shared-GPU mode: the
        # ranks time-slice one GPU and its link, so each gather runs alone)
        peak = min(p[0] if shared_gpu else p[1] for p in peaks)
        achieved = per_rank_bytes / (tmax / 1e3) / 1e9
        return {"bound": "host_link", "achieved": round(achieved, 2), "peak": round(peak, 2), "unit": "GB/s",
                "frac": round(achieved / peak, 3), "traffic": None,
                "kernel": "gather_span_kernel (the worker's own misses: TMA spans + 16-B zero-copy host reads)",
                "algorithmic_bytes_per_launch": int(per_rank_bytes / R),
                "peak_source": f"per-rank pinned 256 MB cudaMemcpy with all {world} ranks copying at once (min over "
                               f"ranks); alone / together per rank: {[[round(a, 2), round(b, 2)] for a, b in peaks]}; "
                               f"rank 0 zero-copy sequential read {round(zc, 2)}; {R} eager steps after the timed "
                               f"region, max over ranks",
                "nvlink": nvl}
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    achieved = 2 * per_rank_bytes / (tmax / 1e3) / 1e9
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(achieved / hbm, 3), "traffic": None,
            "kernel": "gather_span_kernel (the worker's own misses from HBM, read + write)",
            "algorithmic_bytes_per_launch": int(2 * per_rank_bytes / R), "nvlink": nvl}


REF_GB_PER_PROC = {"c1": 0.3, "c2": 2.0, "c3": 4.0, "c5": 4.0}


def run_reference(args, cfg):
    """The reference's CPU implementation of the path (gnnio itself, see
    RefPath) on every host core it can use, on the GPU arms' config. Touches
    neither CUDA nor the product library. Under torchrun only rank 0 runs."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    rp = RefPath(cfg, args, world=world)
    procs = host_procs(REF_GB_PER_PROC.get(args.config, 2.0))
    # the GPU arms time batches W .. W+K-1 after W warm-up batches from a cold
    # cache: the same window here, K rounded up to whole waves of the pool
    K = -(-args.steps // procs) * procs
    W = args.warmup
    rp.run(list(range(W)), procs)
    r = rp.run(list(range(W, W + K)), procs)
    value = r["batches"] / r["seconds"]
    out = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * r["seconds"] / r["batches"], 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64 ids / fp64 priorities / fp32 rows moved",
        "data": (f"synthetic: gnnio.graph.generate_power_law({cfg['n']}, {cfg['avg_degree']}, seed={GRAPH_SEED}, "
                 f"train_fraction={cfg['train']}, num_labels={cfg['labels']}) built on the host by the C "
                 f"restatement oracle/powerlaw_ref.c (bit-identical to gnnio's, tests/test_oracle_golden.py); the "
                 f"same hashed fp32 features; the schedule by gnnio's own ordering"),
        "impl": "reference",
        "config": bench_config(cfg, args, world, rp.col.size, rp.max_degree, len(rp.batches)),
        "feature_gbs": round(r["feature_bytes"] / r["seconds"] / 1e9, 3),
        "timed_batches": r["batches"],
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": procs, "kind": rp.kind,
                         "sample": f"batches {W}..{W + K - 1} of the schedule after {W} warm-up batches from a cold "
                                   f"cache ({K} = --steps rounded up to whole waves of {procs} worker processes): "
                                   f"{rp.what()} sample_batch per batch in a fork pool of {procs} processes, its "
                                   f"FIFO simulate on the persistent state + numpy F[distinct] in batch order in the "
                                   f"main process ({r['cache_gather_s']:.1f}s of {r['seconds']:.1f}s); untimed setup "
                                   f"{rp.setup}"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "isolation": reference_isolation(),
    }
    print(json.dumps(out), flush=True)


def reference_isolation() -> dict:
    """Evidence that the reference arm ran without the product: no product
    module imported, no in-repo shared library mapped, torch (and so CUDA)
    never imported."""
    mapped = set()
    try:
        for line in open("/proc/self/maps"):
            p = line.split()[-1]
            if p.endswith(".so") and p.startswith(ROOT):
                mapped.add(os.path.relpath(p, ROOT))
    except OSError:
        pass
    return {"product_modules": sorted(m for m in sys.modules if m.startswith("paper_2112_08541_b200")),
            "repo_so_mapped": sorted(mapped), "torch_imported": "torch" in sys.modules,
            "reference_package": (import_gnnio() or {}).get("path")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["bgl", "reference"], default="bgl")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--features", choices=["host", "hbm"], default="host")
    ap.add_argument("--graph", choices=["exact", "continuum"], default=None,
                    help="exact: the reference generator's own graph (default for c1/c2); continuum: GPU model (c3)")
    ap.add_argument("--rng", choices=["replay", "counter"], default="replay",
                    help="replay: the reference's numpy stream bit for bit (default); counter: Philox + Floyd")
    ap.add_argument("--order", choices=["proximity", "random"], default="proximity",
                    help="batch ordering: proximity_schedule (BGL, default) or random_shuffle_schedule")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graphs", action="store_true", help="sharded engine: eager steps (no CUDA graphs)")
    ap.add_argument("--sharded", action="store_true", help="use the multi-GPU sharded engine even at N=1")
    ap.add_argument("--exchange", choices=["push", "nccl"], default="push",
                    help="multi-GPU row exchange: home-push over peer memory or NCCL all-to-all")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.graph is None:
        args.graph = "continuum" if args.config in ("c3", "c5") else "exact"
    world = dist_env()[2]
    if args.impl == "reference":
        if "WORLD_SIZE" not in os.environ and args.gpus > 1:
            os.environ["WORLD_SIZE"] = str(args.gpus)      # rank 0 alone runs; the config is the N-GPU one
        run_reference(args, cfg)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch(args.gpus)                                # one process per GPU, as the driver's torchrun
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1 or args.sharded:
        run_sharded(args, cfg)
    else:
        run_bgl(args, cfg)


def relaunch(n: int) -> None:
    """`bench.py --gpus N` without torchrun: re-exec under
    torch.distributed.run with N local ranks (rendezvous on 127.0.0.1),
    exactly as the driver launches N > 1."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


if __name__ == "__main__":
    main()
