"""Cache-capacity x ordering sweep on one B200 (BASELINE.json configs 4/5 shape,
the reference's `compare_policies` / scripts/cache_policy_sweep.py on the
real pipeline): hit %, mini-batches/s and host-miss GB/s of the pipelined
step for proximity vs random ordering.

    python tools/sweep.py --config c2 --caps 0.01,0.02,0.05,0.1,0.2 --steps 150
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
from paper_2112_08541_b200.ordering import random_shuffle_schedule  # noqa: E402
from paper_2112_08541_b200.pipeline import MiniBatchPipeline  # noqa: E402

CONFIGS = dict(bench.CONFIGS)      # c1, c2, c3 (= the C4 sweep's graph), c5


def run(cfg, order, cap, steps, warmup):
    pipe = MiniBatchPipeline(DG, cfg["fanouts"], cfg["b"], order, bench.RUN_SEED,
                             CacheConfig(device_capacity=cap, feature_bytes_per_node=cfg["dim"] * 4), FEATS)
    pipe.capture()
    pipe.reset()
    pipe.prime()
    for _ in range(warmup):
        pipe.step()
    torch.cuda.synchronize()
    c0 = pipe.counters.clone()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        pipe.step()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    d = (pipe.counters - c0).tolist()
    q, hits, miss = d[0], d[1] + d[2] + d[3], d[3] + d[4]
    del pipe
    torch.cuda.empty_cache()
    return {"hit_pct": round(100.0 * hits / max(q, 1), 2), "batches_per_s": round(steps / (ms * 1e-3), 1),
            "rows_per_batch": round(q / steps), "host_miss_gbs": round(miss * cfg["dim"] * 4 / (ms * 1e-3) / 1e9, 2),
            "feature_gbs": round(q * cfg["dim"] * 4 / (ms * 1e-3) / 1e9, 2)}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--caps", default="0.01,0.02,0.05,0.1,0.2")
    ap.add_argument("--steps", type=int, default=150)
    ap.add_argument("--warmup", type=int, default=40)
    ap.add_argument("--orderings", default="proximity,random")
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    DG, FEATS, prox, setup = bench.build_inputs(cfg, "host", "continuum" if a.config in ("c3", "c5") else "exact")
    rnd_batches = random_shuffle_schedule(DG, cfg["b"], seed=bench.RUN_SEED).batches
    rnd = torch.from_numpy(np.concatenate(rnd_batches).astype(np.int32)).cuda()
    out = {"config": a.config, "workload": cfg["workload"], "csr_entries": DG.num_edges, "setup": setup, "rows": []}
    for frac in [float(x) for x in a.caps.split(",")]:
        cap = int(frac * cfg["n"])
        for name, order in (("proximity", prox), ("random", rnd)):
            if name not in a.orderings.split(","):
                continue
            r = run(cfg, order, cap, a.steps, a.warmup)
            r.update(ordering=name, cache_frac=frac, cache_rows=cap)
            out["rows"].append(r)
            print(json.dumps(r), flush=True)
    print(json.dumps(out))
