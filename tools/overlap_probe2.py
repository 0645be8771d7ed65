"""Event timeline of the two branches of a pipelined step (diagnostic)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2112_08541_b200.cachesim import CacheConfig  # noqa: E402
from paper_2112_08541_b200.pipeline import MiniBatchPipeline  # noqa: E402

feat = sys.argv[1] if len(sys.argv) > 1 else "host"
ctas = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = bench.CONFIGS["c2"]
dg, feats, order, _ = bench.build_inputs(cfg, feat)
pipe = MiniBatchPipeline(dg, cfg["fanouts"], cfg["b"], order, 1,
                         CacheConfig(device_capacity=240000, feature_bytes_per_node=400), feats, sampler_ctas=ctas)
for _ in range(30):
    pipe.step_eager()
torch.cuda.synchronize()
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
for it in range(5):
    parity = pipe.k % 2
    t0 = E()
    t0.record()
    cur = torch.cuda.current_stream()
    pipe.s_stream.wait_stream(cur)
    pipe.c_stream.wait_stream(cur)
    s0, s1, c0, c1 = E(), E(), E(), E()
    with torch.cuda.stream(pipe.c_stream):
        c0.record()
        pipe._cache(parity, stream=pipe.c_stream)
        c1.record()
    with torch.cuda.stream(pipe.s_stream):
        s0.record()
        pipe._sample(1 - parity, stream=pipe.s_stream)
        s1.record()
    cur.wait_stream(pipe.s_stream)
    cur.wait_stream(pipe.c_stream)
    pipe.k += 1
    torch.cuda.synchronize()
    print(f"sample [{t0.elapsed_time(s0):.3f}, {t0.elapsed_time(s1):.3f}]  cache [{t0.elapsed_time(c0):.3f}, {t0.elapsed_time(c1):.3f}]")
