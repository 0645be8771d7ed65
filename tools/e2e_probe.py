"""Where does the host-fed (e2e) loop lose vs the device-fed one? Variants of
the bench's e2e loop on C2 host features (diagnostic)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2112_08541_b200.cachesim import CacheConfig  # noqa: E402
from paper_2112_08541_b200.pipeline import MiniBatchPipeline  # noqa: E402

cfg = bench.CONFIGS["c2"]
dg, feats, order, _ = bench.build_inputs(cfg, "host")
b = cfg["b"]
pipe = MiniBatchPipeline(dg, cfg["fanouts"], b, order, 1, CacheConfig(device_capacity=240000, feature_bytes_per_node=400),
                         feats)
pipe.step_eager()
torch.cuda.synchronize()
pipe.capture()
pipe.capture(fed=True)
order_host = order.cpu().numpy().astype(np.int32)
nbl = pipe.num_batches
seeds_pinned = torch.from_numpy(order_host).pin_memory()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def feed(i):
    lo, hi = (i % nbl) * b, min((i % nbl + 1) * b, order_host.size)
    return pipe.feed(i, seeds_pinned[lo:hi])


def run(name, fed, do_flush, wait_copy, steps=120):
    pipe.reset()
    pipe.prime(fed=fed, feed=feed if fed else None)
    for k in range(20):
        if fed:
            feed(k + pipe.lookahead)
        pipe.step(fed=fed)
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream()
    evs = []
    for k in range(20, 20 + steps):
        if do_flush:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pipe.step(fed=fed)
        if fed:
            feed(k + 1 + pipe.lookahead)
            if wait_copy:
                cur.wait_event(pipe.fed_ready[(k + 1 + pipe.lookahead) % len(pipe.fed_ready)])
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    t = statistics.mean(a.elapsed_time(c) for a, c in evs)
    print(f"{name:40s} {1e3 / t:8.1f} b/s", flush=True)


run("device-fed, flush", False, True, False)
run("host-fed, flush, wait copy (bench)", True, True, True)
run("host-fed, flush, no wait", True, True, False)
run("host-fed, no flush, wait copy", True, False, True)
run("device-fed, no flush", False, False, False)
