"""Drive a few eager pipeline steps at a bench config for ncu.

    ncu ... python tools/profile_step.py [--config c2] [--steps 6]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2112_08541_b200.cachesim import CacheConfig  # noqa: E402
from paper_2112_08541_b200.pipeline import MiniBatchPipeline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--features", default="host")
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--warm", type=int, default=20)
ap.add_argument("--rng", default="replay")
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
dg, feats, order, _ = bench.build_inputs(cfg, a.features)
pipe = MiniBatchPipeline(dg, cfg["fanouts"], cfg["b"], order, bench.RUN_SEED,
                         CacheConfig(device_capacity=int(cfg["cache_frac"] * cfg["n"]),
                                     feature_bytes_per_node=cfg["dim"] * 4), feats, rng=a.rng)
pipe.capture()
for _ in range(a.warm):          # graph replays: warm cache (ncu does not see these as separate kernels)
    pipe.step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
miss_rows = []
for _ in range(a.steps):
    k = pipe.k
    pipe.step_eager()
    torch.cuda.synchronize()
    miss_rows.append(int(pipe.miss_count[(k + 1) % len(pipe.miss_count)].item()))   # rows of miss(k+1)
torch.cuda.cudart().cudaProfilerStop()
print("profiled", a.steps, "steps; counters", pipe.counters.tolist())
print("miss-gather rows per profiled step", miss_rows, "row bytes", cfg["dim"] * 4)
