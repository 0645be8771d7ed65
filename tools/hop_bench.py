"""Sampler-only timing and digest at a bench config (A/B of sampler variants).

    BGL_SAMPLER=seg python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/hop_seg.json
    python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/hop_slice.json

Runs the reference-replay sampler (BatchSampler, frontiers + parent indices
kept) on the bench's proximity schedule, one batch after another on one
stream, and records per hop the CUDA-event time of its launches (sampling
kernels incl. prep / heavy; host-synchronous per batch, so launch gaps are
included), the back-to-back time per batch (all hops + dedup, no host sync
between batches) and per batch a SHA-256 digest of every hop's
frontier, parent indices and the distinct set: two variants are bit-identical
when their digests agree (the GPU tests pin one of them to the reference).
"""
import argparse
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2112_08541_b200.ordering import proximity_schedule_device  # noqa: E402
from paper_2112_08541_b200.sampler import BatchSampler, pcg_states, pcg_tables  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--batches", type=int, default=40)
ap.add_argument("--warm", type=int, default=5)
ap.add_argument("--out", default=None)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
dg = bench.make_graph(cfg, "exact" if a.config in ("c1", "c2") else "continuum")
order, _ = proximity_schedule_device(dg, cfg["S"], cfg["b"], seed=bench.RUN_SEED)
order = order.to(torch.int32)
b = cfg["b"]
nb = min(a.batches, order.numel() // b)
tables = pcg_tables(pcg_states(bench.RUN_SEED, range(nb)))
smp = BatchSampler(dg, cfg["fanouts"], b)
H = smp.H
ev = [torch.cuda.Event(enable_timing=True) for _ in range(H + 2)]
hop_ms = [[] for _ in range(H)]
dedup_ms = []
digests = []
for i in range(nb):
    smp.load_seeds(order[i * b:(i + 1) * b])
    torch.cuda.synchronize()
    ev[0].record()
    smp.run(tables[i], hooks=lambda h: ev[h + 1].record())
    ev[H + 1].record()
    torch.cuda.synchronize()
    if i >= a.warm:
        for h in range(H):
            hop_ms[h].append(ev[h].elapsed_time(ev[h + 1]))
        dedup_ms.append(ev[H].elapsed_time(ev[H + 1]))
    counts = smp.host_counts()
    m = hashlib.sha256()
    for h in range(H):
        m.update(smp.frontier(h, counts).cpu().numpy().tobytes())
        m.update(smp.parent_idx(h, counts).cpu().numpy().tobytes())
    m.update(smp.distinct().cpu().numpy().tobytes())
    digests.append(m.hexdigest()[:16])
# timing pass: every batch enqueued back to back (no host sync between
# batches, so launch latency hides behind the GPU), one event pair around it
reps = 3
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
t0.record()
for _ in range(reps):
    for i in range(nb):
        smp.load_seeds(order[i * b:(i + 1) * b])
        smp.run(tables[i])
t1.record()
torch.cuda.synchronize()
batch_us = 1e3 * t0.elapsed_time(t1) / (reps * nb)
# per-hop time, warm: one batch's hop h (all of its launches) captured in a
# CUDA graph and replayed back to back (inputs unchanged between replays)
hop_graph_us = []
i = nb - 1
smp.load_seeds(order[i * b:(i + 1) * b])
smp.run(tables[i])
torch.cuda.synchronize()
side = torch.cuda.Stream()
for h in range(H):
    g = torch.cuda.CUDAGraph()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        smp.run(tables[i], hops=range(h, h + 1), dedup=False)     # warm-up outside the graph
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=side):
            smp.run(tables[i], hops=range(h, h + 1), dedup=False)
    torch.cuda.synchronize()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    t0.record()
    for _ in range(200):
        g.replay()
    t1.record()
    torch.cuda.synchronize()
    hop_graph_us.append(round(1e3 * t0.elapsed_time(t1) / 200, 2))
smp.clear_marks()
rep = {"config": a.config, "sampler_us_per_batch": round(batch_us, 2), "hop_graph_us": hop_graph_us, "sampler": os.environ.get("BGL_SAMPLER", "default"),
       "slice_draws": os.environ.get("BGL_SLICE_DRAWS", "auto"), "batches": nb, "timed": nb - a.warm,
       "hop_us_mean": [round(1e3 * float(np.mean(x)), 2) for x in hop_ms],
       "hop_us_min": [round(1e3 * float(np.min(x)), 2) for x in hop_ms],
       "dedup_us_mean": round(1e3 * float(np.mean(dedup_ms)), 2),
       "digest": hashlib.sha256("".join(digests).encode()).hexdigest()[:16], "batch_digests": digests}
print(json.dumps({k: v for k, v in rep.items() if k != "batch_digests"}))
if a.out:
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(rep, open(a.out, "w"))
