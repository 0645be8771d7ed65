"""Per-branch timeline of the pipelined step (diagnostics).

    python tools/branch_timeline.py [--config c2] [--features hbm] [--steps 20]

Runs eager pipelined steps behind a GPU-side gate (torch.cuda._sleep on the
launching stream), so every branch is enqueued before any of them starts and
the CUDA events around each branch show the GPU's own overlap, not the
host's launch order: per branch (back, miss, LI, sample b = last hop + dedup,
sample a = staging + first hops) the mean start and end relative to the step
start, and the step's span.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2112_08541_b200.cachesim import CacheConfig  # noqa: E402
from paper_2112_08541_b200.pipeline import MiniBatchPipeline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--features", default="hbm")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--warm", type=int, default=20)
ap.add_argument("--out", default=None)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
dg, feats, order, _ = bench.build_inputs(cfg, a.features)
pipe = MiniBatchPipeline(dg, cfg["fanouts"], cfg["b"], order, bench.RUN_SEED,
                         CacheConfig(device_capacity=int(cfg["cache_frac"] * cfg["n"]),
                                     feature_bytes_per_node=cfg["dim"] * 4), feats)
pipe.capture()
for _ in range(a.warm):
    pipe.step()
torch.cuda.synchronize()

names = ["back", "miss", "li", "sample_b", "sample_a"]
marks = {}


def wrap(name, fn):
    def w(*args, **kw):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(*args, **kw)
        e1.record()
        marks[name] = (e0, e1)
    return w


orig = {"_back": pipe._back, "_miss": pipe._miss, "_li": pipe._li, "_sample": pipe._sample}
pipe._back = wrap("back", orig["_back"])
pipe._miss = wrap("miss", orig["_miss"])
pipe._li = wrap("li", orig["_li"])


def sample(batch, stream=None, fed=False, hooks=None, part="all"):
    wrap("sample_" + part, orig["_sample"])(batch, stream=stream, fed=fed, hooks=hooks, part=part)


pipe._sample = sample
rows = {n: [] for n in names}
span = []
for _ in range(a.steps):
    marks.clear()
    torch.cuda._sleep(3_000_000)          # gate: the whole step is enqueued before it starts
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    pipe.step_eager()
    t1.record()
    torch.cuda.synchronize()
    span.append(1e3 * t0.elapsed_time(t1))
    for n in names:
        if n in marks:
            e0, e1 = marks[n]
            rows[n].append((1e3 * t0.elapsed_time(e0), 1e3 * t0.elapsed_time(e1)))
rep = {"config": a.config, "features": a.features, "steps": a.steps,
       "step_us_mean": round(float(np.mean(span)), 2),
       "branches_us": {n: {"start": round(float(np.mean([r[0] for r in v])), 2),
                           "end": round(float(np.mean([r[1] for r in v])), 2)} for n, v in rows.items() if v}}
print(json.dumps(rep))
if a.out:
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(rep, open(a.out, "w"))
