"""Papers100M-shaped proximity schedule: device vs the numpy oracle (equality + times)."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench
from oracle import ordering_oracle as oo
from paper_2112_08541_b200.ordering import proximity_schedule_device
cfg = bench.CONFIGS["c3"]
dg = bench.make_graph(cfg, "continuum")
t = time.time(); order, _ = proximity_schedule_device(dg, cfg["S"], cfg["b"], seed=bench.RUN_SEED); torch.cuda.synchronize(); print("device", time.time() - t, flush=True)
off = dg.indptr.cpu().numpy(); col = dg.indices.cpu().numpy(); tm = dg.train_mask.cpu().numpy()
t = time.time()
sched = oo.proximity_schedule(off, col, tm, cfg["S"], cfg["b"], bench.RUN_SEED)
print("oracle", time.time() - t, flush=True)
flat = np.concatenate(sched) if isinstance(sched, list) else np.concatenate(sched.batches)
print("equal", np.array_equal(flat, order.cpu().numpy()), flat.size)
