"""cProfile of the gnnio-signature drop-in calls at the C2 bench shape.

    python tools/profile_dropin.py [--batches 25]

Builds the bench's C2 inputs, then profiles sampler.simulate_epoch,
FeatureCacheEngine.retrieve and cachesim.simulate over the same trace (the
bench's `e2e_dropin` window) and prints the top host-side costs of each.
"""
import argparse
import cProfile
import io
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2112_08541_b200.cachesim import CacheConfig, simulate  # noqa: E402
from paper_2112_08541_b200.features import FeatureCacheEngine  # noqa: E402
from paper_2112_08541_b200.ordering import BatchSchedule  # noqa: E402
from paper_2112_08541_b200.sampler import SamplingConfig, simulate_epoch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", type=int, default=25)
ap.add_argument("--features", default="host")
a = ap.parse_args()
cfg = bench.CONFIGS["c2"]
dg, feats, order, _ = bench.build_inputs(cfg, a.features)
b = cfg["b"]
oh = order.cpu().numpy()
sched = BatchSchedule(batches=[oh[i * b:(i + 1) * b].astype(np.int64) for i in range(a.batches)], batch_size=b,
                      policy="proximity")
scfg = SamplingConfig(fanouts=tuple(cfg["fanouts"]), batch_size=b, seed=bench.RUN_SEED)
ccfg = CacheConfig(device_capacity=int(cfg["cache_frac"] * cfg["n"]), feature_bytes_per_node=cfg["dim"] * 4)
simulate_epoch(dg, None, BatchSchedule(batches=sched.batches[:2], batch_size=b, policy="proximity"), scfg)
torch.cuda.synchronize()


def prof(name, fn):
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    out = fn()
    torch.cuda.synchronize()
    pr.disable()
    dt = time.perf_counter() - t0
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(14)
    print(f"== {name}: {1e3 * dt / a.batches:.3f} ms per batch")
    print("\n".join(s.getvalue().splitlines()[:34]))
    return out


trace, _ = prof("simulate_epoch", lambda: simulate_epoch(dg, None, sched, scfg))
eng = FeatureCacheEngine(ccfg, feats, max(x.size for x in trace.batches))
prof("retrieve", lambda: [eng.retrieve(ids, i) for i, ids in enumerate(trace.batches)])
prof("simulate (cold)", lambda: simulate(trace, ccfg))
prof("simulate (again)", lambda: simulate(trace, ccfg))
