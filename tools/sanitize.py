"""Drive every kernel family once on small inputs (for compute-sanitizer):
    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize.py
sampler (replay + counter), dedup/relabel, FIFO lookup/insert (pipeline,
eager steps, host + HBM features, span and per-row miss gathers), static warm,
BFS ordering + interleave, shuffling TV, partition/scatter, native generator;
round 2: sparse-ID hash dedup + ring remap, LRU / LFU updates (every level
kind, sparse IDs), the sampler timeline trace."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2112_08541_b200 as bgl  # noqa: E402
from paper_2112_08541_b200.cachesim import CacheConfig  # noqa: E402
from paper_2112_08541_b200.distributed import GpuShardOps  # noqa: E402
from paper_2112_08541_b200.features import synthetic_features  # noqa: E402
from paper_2112_08541_b200.graph import generate_power_law_exact_device  # noqa: E402
from paper_2112_08541_b200.ordering import proximity_schedule_device  # noqa: E402
from paper_2112_08541_b200.pipeline import MiniBatchPipeline  # noqa: E402

dg = generate_power_law_exact_device(6000, 12, seed=2, train_fraction=0.3, num_labels=4)
hg = dg.to_host()
order, _ = proximity_schedule_device(dg, 3, 128, seed=1)
for rng in ("replay", "counter"):
    for where in ("host", "hbm"):
        feats = synthetic_features(6000, 32, seed=1, device_resident=(where == "hbm"))
        pipe = MiniBatchPipeline(dg, (10, 5), 128, order, 3, CacheConfig(device_capacity=500, feature_bytes_per_node=128),
                                 feats, rng=rng)
        for _ in range(6):
            pipe.step_eager()
        pipe.engine.miss_spans = False
        for _ in range(3):
            pipe.step_eager()
        torch.cuda.synchronize()
sys.path.insert(0, os.path.join(ROOT, "tests"))
import sampler_paths  # noqa: E402

g_hub, seeds_hub = sampler_paths.inputs(num_seeds=600)     # hub parents inside runs (heavy gaps, CTA kernel)
for f in ((5, 5), (32,)):
    bgl.sample_batch(g_hub, seeds_hub, bgl.SamplingConfig(fanouts=f, seed=9), batch_seed=3)
bgl.sampler.sample_batch_relabelled(hg, hg.train_nodes()[:64], bgl.SamplingConfig(fanouts=(5, 3), seed=1))
sched = bgl.proximity_schedule(hg, 2, 100, seed=1)
trace, _ = bgl.simulate_epoch(hg, None, sched, bgl.SamplingConfig(fanouts=(4, 2), seed=1))
bgl.simulate(trace, CacheConfig(device_capacity=300, host_capacity=50, num_devices=2))
bgl.simulate(trace, CacheConfig(device_capacity=300, num_devices=2, policy="static-degree"), g=hg)
bgl.shuffling_error(sched, hg.labels)
ops = GpuShardOps(4, 2000, 128)
ids = torch.unique(torch.randint(0, 6000, (1500,), device="cuda")).to(torch.int32)
part, pos, counts = ops.partition(ids)
ops.scatter(pos, torch.zeros((len(ids), 32), device="cuda"), torch.zeros((len(ids), 32), device="cuda"))
# round 2: sparse int64 IDs (hash dedup, home map, remap) on FIFO / LRU / LFU, static; the timeline trace
from paper_2112_08541_b200.sampler import AccessTrace  # noqa: E402
rng = np.random.default_rng(4)
universe = np.unique(rng.integers(2**33, 2**40, size=300))
for policy in ("fifo", "lru", "lfu"):
    cfg = CacheConfig(device_capacity=40, host_capacity=25, num_devices=3, policy=policy)
    st = bgl.cachesim.cold_state(cfg)
    for k in range(3):
        part = [rng.choice(universe[: 100 * (k + 1)], size=70) for _ in range(3)]
        bgl.simulate(AccessTrace(batches=part), cfg, state=st, record_outcomes=True)
    bgl.simulate(trace, CacheConfig(device_capacity=200, host_capacity=60, num_devices=2, policy=policy))
from paper_2112_08541_b200 import _lib  # noqa: E402
buf = torch.zeros(8 + 8 * 4096, dtype=torch.int64, device="cuda")
_lib.check(_lib.load().bgl_debug_seg_trace(buf.data_ptr()))
bgl.sample_batch(g_hub, seeds_hub, bgl.SamplingConfig(fanouts=(5, 5), seed=9), batch_seed=4)
torch.cuda.synchronize()
_lib.check(_lib.load().bgl_debug_seg_trace(None))
torch.cuda.synchronize()
print("sanitize driver done")
