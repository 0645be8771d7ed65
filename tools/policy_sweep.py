"""Cache-policy x capacity x ordering sweep through the drop-in API at the
products shape -- the reference's scripts/cache_policy_sweep.py (every
policy of POLICIES, proximity vs random ordering) on the GPU, with the
per-batch simulate time and the amortized update operations of every cell
(cachesim.amortized_update_ops, cachesim.py:366-375).

    python tools/policy_sweep.py [--config c2] [--batches 188] [--out gpurun_out/policy_sweep_c2.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2112_08541_b200.cachesim import POLICIES, CacheConfig, amortized_update_ops, simulate  # noqa: E402
from paper_2112_08541_b200.ordering import BatchSchedule, random_shuffle_schedule  # noqa: E402
from paper_2112_08541_b200.sampler import SamplingConfig, simulate_epoch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--batches", type=int, default=188)
ap.add_argument("--caps", default="0.01,0.02,0.05,0.1,0.2")
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "policy_sweep.json"))
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
dg, _, order, _ = bench.build_inputs(cfg, "hbm")
hg = dg.to_host()
b = cfg["b"]
oh = order.cpu().numpy().astype(np.int64)
nb = min(a.batches, -(-oh.size // b))
scfg = SamplingConfig(fanouts=tuple(cfg["fanouts"]), batch_size=b, seed=bench.RUN_SEED)
scheds = {"proximity": BatchSchedule(batches=[oh[i * b:(i + 1) * b] for i in range(nb)], batch_size=b,
                                     policy="proximity"),
          "random": random_shuffle_schedule(hg, b, seed=bench.RUN_SEED)}
scheds["random"].batches = scheds["random"].batches[:nb]
traces = {}
for name, sc in scheds.items():
    t0 = time.perf_counter()
    traces[name] = simulate_epoch(dg, None, sc, scfg)[0]
    print(f"trace {name}: {nb} batches, {np.mean([x.size for x in traces[name].batches]):.0f} distinct per batch, "
          f"{time.perf_counter() - t0:.2f} s", flush=True)
rows = []
for policy in POLICIES:
    for ordering, trace in traces.items():
        for f in (float(x) for x in a.caps.split(",")):
            cap = int(f * cfg["n"])
            c = CacheConfig(device_capacity=cap, policy=policy, feature_bytes_per_node=cfg["dim"] * 4)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = simulate(trace, c, g=dg)
            dt = time.perf_counter() - t0
            am = amortized_update_ops(rep)
            row = {"policy": policy, "ordering": ordering, "cache_frac": f, "capacity": cap,
                   "hit_ratio": round(rep.hit_ratio, 6), "simulate_ms_per_batch": round(1e3 * dt / nb, 3),
                   **{k: round(v, 1) for k, v in am.items()}}
            rows.append(row)
            print(row, flush=True)
os.makedirs(os.path.dirname(a.out), exist_ok=True)
json.dump({"config": a.config, "workload": bench.workload_text(cfg, "hbm"), "batches": nb,
           "source": "tools/policy_sweep.py: cachesim.simulate (drop-in API) on traces from sampler.simulate_epoch",
           "rows": rows}, open(a.out, "w"), indent=1)
