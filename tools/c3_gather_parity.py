"""Papers100M-shaped gather parity: the bench's C3 pipeline (57 GB of pinned
host features, FIFO cache of 11.1M rows in HBM, CUDA-graph steps) -- every row
of the checked batches equals the regenerated feature row F[id] (the hashed
features of oracle/features_oracle.py), and the distinct set equals the
oracle sampler's for the same batch.
    python tools/c3_gather_parity.py [--features host|hbm] [--steps 40]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from oracle import features_oracle as fo  # noqa: E402
from oracle import sampler_oracle as so  # noqa: E402
from paper_2112_08541_b200.cachesim import CacheConfig  # noqa: E402
from paper_2112_08541_b200.pipeline import MiniBatchPipeline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--features", default="host")
ap.add_argument("--steps", type=int, default=40)
a = ap.parse_args()
cfg = bench.CONFIGS["c3"]
dg, feats, order, setup = bench.build_inputs(cfg, a.features, "continuum")
pipe = MiniBatchPipeline(dg, cfg["fanouts"], cfg["b"], order, bench.RUN_SEED,
                         CacheConfig(device_capacity=int(cfg["cache_frac"] * cfg["n"]),
                                     feature_bytes_per_node=cfg["dim"] * 4), feats)
pipe.capture()
off, col = dg.indptr.cpu().numpy(), dg.indices.cpu().numpy()
order_h = order.cpu().numpy().astype(np.int64)
b = cfg["b"]
checked = rows_checked = 0
t0 = time.time()
for step in range(a.steps):
    pipe.step()
    if step % 8 == 7:                       # batch `step` is complete after this step
        torch.cuda.synchronize()
        i = pipe.last_batch()
        ids = pipe.distinct().cpu().numpy()
        rows = pipe.rows().cpu().numpy()
        assert np.array_equal(rows, fo.synthetic_features(ids, cfg["dim"], seed=bench.GRAPH_SEED)), i
        _, _, d_o, _ = so.sample_batch(off, col, order_h[i * b:(i + 1) * b], cfg["fanouts"], bench.RUN_SEED, i)
        assert np.array_equal(ids, d_o), i
        checked += 1
        rows_checked += ids.size
print(f"C3 {a.features}: {checked} batches, {rows_checked} rows equal F[id]; distinct sets equal the oracle's; "
      f"counters {pipe.counters.tolist()}; {time.time() - t0:.1f} s; setup {setup}")
