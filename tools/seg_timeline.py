"""Per-run timeline of the segmented sampler walk (diagnostics).

    python tools/seg_timeline.py [--config c2] [--features hbm] [--out gpurun_out/seg_timeline.json]

Warms the bench pipeline with graph replays, then runs one eager step with
`bgl_debug_seg_trace` on: every run of `sample_seg_kernel` records
{parents, run, SM, walk draws, t_claim, t_walk, t_post, t_end} (globaltimer).
Prints per hop: kernel span, run durations (setup / walk / post), how many
runs start after the first wave, and the busy-warp profile over time.
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
from paper_2112_08541_b200 import _lib  # noqa: E402
from paper_2112_08541_b200.cachesim import CacheConfig  # noqa: E402
from paper_2112_08541_b200.pipeline import MiniBatchPipeline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--features", default="hbm")
ap.add_argument("--warm", type=int, default=20)
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "seg_timeline.json"))
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
cap = 1 << 20
W = 16   # words per record (csrc/sampler.cu kSegTraceWords)
buf = torch.zeros(W + W * cap, dtype=torch.int64, device="cuda")
lib = _lib.load()
_lib.check(lib.bgl_debug_seg_trace(buf.data_ptr()))
pipe.step_eager()
torch.cuda.synchronize()
_lib.check(lib.bgl_debug_seg_trace(None))
nrec = int(buf[0].item())
rec = buf[W:W + W * nrec].view(nrec, W).cpu().numpy()
report = {"config": a.config, "features": a.features, "hops": []}
for n in sorted(set(rec[:, 0].tolist())):
    r = rec[rec[:, 0] == n]
    t0 = r[:, 4].min()
    claim, walk, post, end = (r[:, 4] - t0) / 1e3, (r[:, 5] - t0) / 1e3, (r[:, 6] - t0) / 1e3, (r[:, 7] - t0) / 1e3
    span = end.max()
    setup_us, walk_us, post_us = walk - claim, post - walk, end - post
    loaded, prefix = (r[:, 8] - t0) / 1e3, (r[:, 9] - t0) / 1e3
    draws = r[:, 3].astype(np.float64)
    # busy runs over time (1 us bins)
    bins = np.arange(0, span + 1.0, 1.0)
    busy = [int(((claim <= b) & (end > b)).sum()) for b in bins]
    late = int((claim > 0.25 * span).sum())
    h = {"parents": int(n), "runs": int(len(r)), "span_us": round(float(span), 2),
         "setup_us_mean": round(float(setup_us.mean()), 2),
         "setup_split_us_mean": {"loads": round(float((loaded - claim).mean()), 2),
                                 "lookback": round(float((prefix - loaded).mean()), 2),
                                 "layout": round(float((walk - prefix).mean()), 2)},
         "lookback_us_p50_p90_max": [round(float(np.percentile(prefix - loaded, q)), 2) for q in (50, 90, 100)],
         "walk_us_mean": round(float(walk_us.mean()), 2),
         "post_us_mean": round(float(post_us.mean()), 2), "run_us_mean": round(float((end - claim).mean()), 2),
         "run_us_p50_p90_max": [round(float(np.percentile(end - claim, q)), 2) for q in (50, 90, 100)],
         "draws_mean": round(float(draws.mean()), 1), "draws_p90_max": [float(np.percentile(draws, 90)), float(draws.max())],
         "walk_ns_per_draw": round(float((walk_us * 1e3).sum() / max(draws.sum(), 1)), 3),
         "runs_claimed_after_25pct_of_span": late,
         "claim_us_p50_p99_max": [round(float(np.percentile(claim, q)), 2) for q in (50, 99, 100)],
         "end_us_p10_p50_p90": [round(float(np.percentile(end, q)), 2) for q in (10, 50, 90)],
         "busy_runs_per_us": busy}
    report["hops"].append(h)
    print({k: v for k, v in h.items() if k != "busy_runs_per_us"})
    print("  busy runs every 5 us:", busy[::5])
os.makedirs(os.path.dirname(a.out), exist_ok=True)
json.dump(report, open(a.out, "w"))
