"""Event timeline of the three branches of a pipelined step (diagnostic)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2112_08541_b200.cachesim import CacheConfig  # noqa: E402
from paper_2112_08541_b200.pipeline import MiniBatchPipeline  # noqa: E402

feat = sys.argv[1] if len(sys.argv) > 1 else "host"
mode = sys.argv[2] if len(sys.argv) > 2 else "all"
cfg = bench.CONFIGS["c2"]
dg, feats, order, _ = bench.build_inputs(cfg, feat)
pipe = MiniBatchPipeline(dg, cfg["fanouts"], cfg["b"], order, 1,
                         CacheConfig(device_capacity=240000, feature_bytes_per_node=400), feats)
for _ in range(30):
    pipe.step_eager()
torch.cuda.synchronize()
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
for it in range(6):
    k = pipe.k
    t0 = E()
    t0.record()
    cur = torch.cuda.current_stream()
    sb, sf, ss = pipe.streams
    for s in pipe.streams:
        s.wait_stream(cur)
    ev = {n: E() for n in ("f0", "f1", "f2", "s0", "s1", "b0", "b1")}
    with torch.cuda.stream(sf):
        ev["f0"].record()
        pipe._front(k + 1, stream=sf, events=[ev["f1"]])
        ev["f2"].record()
    if mode in ("all", "fs"):
        with torch.cuda.stream(ss):
            ev["s0"].record()
            pipe._sample(k + 2, stream=ss)
            ev["s1"].record()
    if mode in ("all", "fb"):
        with torch.cuda.stream(sb):
            ev["b0"].record()
            pipe._back(k, stream=sb)
            ev["b1"].record()
    for s in pipe.streams:
        cur.wait_stream(s)
    pipe.k += 1
    if mode not in ("all", "fs"):
        with torch.cuda.stream(ss):
            pipe._sample(k + 2, stream=ss)
    if mode not in ("all", "fb"):
        with torch.cuda.stream(sb):
            pipe._back(k, stream=sb)
    torch.cuda.synchronize()
    f = lambda a: t0.elapsed_time(ev[a])  # noqa: E731
    line = f"front [{f('f0'):.3f} lookup/insert->{f('f1'):.3f} miss->{f('f2'):.3f}]"
    if mode in ("all", "fs"):
        line += f"  sample [{f('s0'):.3f}, {f('s1'):.3f}]"
    if mode in ("all", "fb"):
        line += f"  back [{f('b0'):.3f}, {f('b1'):.3f}]"
    print(mode, line, flush=True)
