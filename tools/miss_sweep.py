"""Sweep the host-link miss gather variants on the bench workload (C2, host
features): serialised per-stage events of pipeline steps, miss-gather time and
algorithmic GB/s per variant. Run under gpurun on one GPU."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2112_08541_b200.cachesim import CacheConfig  # noqa: E402
from paper_2112_08541_b200.pipeline import MiniBatchPipeline  # noqa: E402

cfg = bench.CONFIGS[os.environ.get("CFG", "c2")]
dg, feats, order, _ = bench.build_inputs(cfg, "host")
rb = cfg["dim"] * 4
pipe = MiniBatchPipeline(dg, cfg["fanouts"], cfg["b"], order, bench.RUN_SEED,
                         CacheConfig(device_capacity=int(cfg["cache_frac"] * cfg["n"]), feature_bytes_per_node=rb),
                         feats)
peak = bench.host_link_peak_gbs()
variants = [("mode2", 74, 4)] + [("list", c, r) for c in (74, 148, 296) for r in (2, 4, 8)]
res = []
for name, ctas, rows in variants:
    pipe.compact_misses = name == "list"
    pipe.engine.miss_ctas = ctas
    pipe.engine.miss_rows_in_flight = rows
    pipe.reset()
    for _ in range(25):
        pipe.step_eager()
    torch.cuda.synchronize()
    hist, ms, by = [], [], []
    for _ in range(12):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
        cb = pipe.counters.clone()
        pipe.step_serial(evs)
        torch.cuda.synchronize()
        hist.append((pipe.counters - cb).cpu().tolist())
        if len(hist) >= 2:
            ca = hist[-2]
            by.append((ca[3] + ca[4]) * rb)
            ms.append(evs[3].elapsed_time(evs[4]))
    gbs = [b / (m * 1e-3) / 1e9 for b, m in zip(by, ms)]
    # pipelined throughput with this variant (graph replays)
    pipe.graphs.clear()
    pipe.reset()
    pipe.capture()
    pipe.reset()
    pipe.prime()
    for _ in range(20):
        pipe.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(150):
        pipe.step()
    e1.record()
    torch.cuda.synchronize()
    bps = 150 / (e0.elapsed_time(e1) * 1e-3)
    r = {"variant": name, "ctas": ctas, "rows_in_flight": rows, "miss_ms": round(statistics.mean(ms), 4),
         "miss_alg_gbs": round(statistics.mean(gbs), 2), "frac": round(statistics.mean(gbs) / peak, 3),
         "pipelined_batches_per_s": round(bps, 1)}
    print(json.dumps(r), flush=True)
    res.append(r)
print(json.dumps({"host_link_peak_gbs": round(peak, 2)}))
