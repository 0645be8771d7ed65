"""Pipelined step time vs the host-link floor (sum of miss-gather times) over the
same batches from the same cold cache (diagnostic)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2112_08541_b200.cachesim import CacheConfig  # noqa: E402
from paper_2112_08541_b200.pipeline import MiniBatchPipeline  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
N = 120
dg, feats, order, _ = bench.build_inputs(cfg, "host")
pipe = MiniBatchPipeline(dg, cfg["fanouts"], cfg["b"], order, 1,
                         CacheConfig(device_capacity=int(0.1 * cfg["n"]), feature_bytes_per_node=cfg["dim"] * 4), feats)
pipe.capture()
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
# serial pass: per-stage times for steps 0..N-1
pipe.reset()
pipe.prime()
tot = [0.0] * 6
for _ in range(N):
    ev = [E() for _ in range(7)]
    pipe.step_serial(ev)
    torch.cuda.synchronize()
    for i in range(6):
        tot[i] += ev[i].elapsed_time(ev[i + 1])
print("serial stage totals ms (sample, dedup, LI, miss, hit, copy):", [round(t, 2) for t in tot])
# pipelined pass over the same batches
pipe.reset()
pipe.prime()
s, e = E(), E()
s.record()
for _ in range(N):
    pipe.step()
e.record()
torch.cuda.synchronize()
print("pipelined total ms", round(s.elapsed_time(e), 2), "per step", round(s.elapsed_time(e) / N, 4),
      "miss floor per step", round(tot[3] / N, 4))
# miss gathers alone, back to back, same batches (cache state replayed by LI)
pipe.reset()
pipe.prime()
s.record()
for k in range(N):
    pipe._li(k + 2)
    pipe._miss(k + 1)
    pipe._back(k)
    pipe._sample(k + 3, part="b")
    pipe._sample(k + 4, part="a")
e.record()
torch.cuda.synchronize()
print("eager serial total ms", round(s.elapsed_time(e), 2))
