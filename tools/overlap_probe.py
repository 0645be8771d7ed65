"""Time the two branches of a pipelined step alone and together (diagnostic)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2112_08541_b200.cachesim import CacheConfig  # noqa: E402
from paper_2112_08541_b200.pipeline import MiniBatchPipeline  # noqa: E402

feat = sys.argv[1] if len(sys.argv) > 1 else "host"
cfg = bench.CONFIGS["c2"]
dg, feats, order, _ = bench.build_inputs(cfg, feat)
ctas = [int(x) for x in sys.argv[2:]] or [0]
for c in ctas:
    pipe = MiniBatchPipeline(dg, cfg["fanouts"], cfg["b"], order, 1,
                             CacheConfig(device_capacity=240000, feature_bytes_per_node=400), feats, sampler_ctas=c)
    pipe.capture()
    for _ in range(30):
        pipe.step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(100):
        pipe.step()
    e.record()
    torch.cuda.synchronize()
    print(feat, "sampler_ctas", c, "graph step ms", s.elapsed_time(e) / 100, flush=True)
    del pipe
sys.exit(0)


def timed(fn, n=50):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


print("graph step      ", timed(pipe.step))
print("eager overlapped", timed(pipe.step_eager))
par = pipe.k % 2
print("sample only     ", timed(lambda: pipe._sample(1 - par)))
print("cache only      ", timed(lambda: pipe._cache(par)))
g = torch.cuda.CUDAGraph()
cs = torch.cuda.Stream()
cs.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(cs):
    with torch.cuda.graph(g, stream=cs):
        pipe._cache(par, stream=cs)
torch.cuda.current_stream().wait_stream(cs)
print("cache graph     ", timed(g.replay))
