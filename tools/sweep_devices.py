"""BASELINE.json configs 4/5 at d = 1/2/4/8 GPUs through the drop-in API
(the reference's `compare_policies` sweep with `num_devices=d`,
cachesim.py:378-409, the node-ID-sharded levels of cachesim.py:319-320):
the trace of the first `--batches` mini-batches of the papers100M-shaped
graph (sampler.simulate_epoch on the device), then `cachesim.compare_policies`
(static-degree and FIFO cells) for every cache fraction and device count,
plus FIFO with random ordering. Hit / peer-hit / miss fractions are exact
results of the reference semantics computed on one B200; throughput at d > 1
needs d GPUs (bench.py --gpus d).

    python tools/sweep_devices.py --config c3 --batches 200 --out profiles/r02/sweep_c4_devices.json
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
from paper_2112_08541_b200.cachesim import CacheConfig, compare_policies, simulate  # noqa: E402
from paper_2112_08541_b200.ordering import BatchSchedule, proximity_schedule_device  # noqa: E402
from paper_2112_08541_b200.sampler import SamplingConfig, simulate_epoch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--batches", type=int, default=200)
ap.add_argument("--fracs", default="0.01,0.02,0.05,0.1,0.2")
ap.add_argument("--devices", default="1,2,4,8")
ap.add_argument("--out", default=None)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
n, b = cfg["n"], cfg["b"]
t0 = time.time()
gen = bench.make_graph(cfg, "continuum" if a.config in ("c3", "c5") else "exact")
torch.cuda.synchronize()
t1 = time.time()
scfg = SamplingConfig(fanouts=tuple(cfg["fanouts"]), batch_size=b, seed=bench.RUN_SEED)
traces = {}
for kind in ("proximity", "random"):
    if kind == "proximity":
        flat, _ = proximity_schedule_device(gen, cfg["S"], b, seed=bench.RUN_SEED)
        flat = flat.cpu().numpy().astype(np.int64)
    else:
        from paper_2112_08541_b200.ordering import _train_ids
        flat = np.random.default_rng(bench.RUN_SEED).permutation(_train_ids(gen)).astype(np.int64)
    sched = BatchSchedule(batches=[flat[i * b:(i + 1) * b] for i in range(a.batches)], batch_size=b, policy=kind)
    ts = time.time()
    trace, _ = simulate_epoch(gen, None, sched, scfg)
    traces[kind] = (trace, time.time() - ts)
t2 = time.time()
fracs = [float(x) for x in a.fracs.split(",")]
rows = []
for d in (int(x) for x in a.devices.split(",")):
    caps = [int(f * n) // d for f in fracs]
    ts = time.time()
    for r in compare_policies(gen, traces["proximity"][0], caps, policies=("static-degree", "fifo"), num_devices=d,
                              feature_bytes_per_node=cfg["dim"] * 4):
        r.update(devices=d, ordering="proximity", cache_frac=fracs[caps.index(r["capacity"])])
        rows.append(r)
    for f, cap in zip(fracs, caps):           # FIFO cells with the peer split, and random ordering
        for kind in ("proximity", "random"):
            rep = simulate(traces[kind][0], CacheConfig(device_capacity=cap, num_devices=d,
                                                        feature_bytes_per_node=cfg["dim"] * 4))
            q = rep.total_queries
            rows.append({"policy": "fifo", "capacity": cap, "devices": d, "ordering": kind, "cache_frac": f,
                         "hit_ratio": rep.hit_ratio, "own_hit_ratio": sum(rep.batch_own_hits) / q,
                         "peer_hit_ratio": sum(rep.batch_peer_hits) / q, "miss_ratio": rep.misses / q,
                         "remote_fetch_gb_per_batch": rep.remote_fetch_bytes / len(rep.batch_queries) / 1e9,
                         "peer_gb_per_batch": rep.peer_bytes / len(rep.batch_queries) / 1e9})
    print(f"d={d}: {time.time() - ts:.1f}s", flush=True)
out = {"config": a.config, "workload": cfg["workload"], "batches": a.batches, "num_nodes": n,
       "csr_entries": gen.num_edges,
       "setup_s": {"graph": round(t1 - t0, 1), "traces": {k: round(v[1], 1) for k, v in traces.items()},
                   "all": round(t2 - t0, 1)},
       "api": "sampler.simulate_epoch (trace) -> cachesim.compare_policies / simulate with num_devices=d",
       "rows": rows}
if a.out:
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
for r in rows:
    if r["policy"] == "fifo" and "own_hit_ratio" in r:
        print(f"d={r['devices']} {r['ordering']:9s} cache {r['cache_frac']:.2f}: hit {100 * r['hit_ratio']:.2f}% "
              f"(peer {100 * r['peer_hit_ratio']:.2f}%), remote {r['remote_fetch_gb_per_batch']:.3f} GB/batch")
