"""GPU test of the peer-push sharded cache (PeerPushFeatureCache): two
processes share one GPU (CUDA IPC between processes works on the same device),
each is home of one shard and worker of every other batch; homes gather rows
and store them straight into the worker's output buffer through the IPC
mapping (bgl_gather_rows_push). The ID exchange goes through gloo on host
tensors. Result must equal the reference's 2-device simulation."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cache_oracle as co
from oracle import features_oracle as fo

pytestmark = pytest.mark.gpu
WORLD = 2


def _worker(rank, port, batches, cap, dim, where, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_2112_08541_b200.distributed import GpuShardEngine, GpuShardOps, PeerPushFeatureCache
    from paper_2112_08541_b200.features import synthetic_features
    n = 20000
    feats = synthetic_features(n, dim, seed=8, device_resident=(where == "hbm"))
    maxb = max(len(b) for b in batches)
    eng = GpuShardEngine(rank, WORLD, cap, feats, maxb)
    ops = GpuShardOps(WORLD, maxb, dim * 4)
    sc = PeerPushFeatureCache(rank, WORLD, eng, ops, dim, maxb, cpu_collectives=True)
    out = {}
    for j in range(len(batches) // WORLD):
        i = j * WORLD + rank
        rows, codes = sc.step(torch.from_numpy(batches[i].astype(np.int32)).cuda())
        out[f"rows{i}"] = rows.cpu().numpy()
        out[f"codes{i}"] = codes.cpu().numpy()
    np.savez(path + f".{rank}.npz", **out)
    dist.barrier()
    sc.close()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("where", ["host", "hbm"])
def test_peer_push_matches_reference_simulation(where):
    rng = np.random.default_rng(12)
    dim, cap = 32, 400
    batches = [np.unique(rng.integers(0, 3000 + 200 * i, size=1500)) for i in range(10)]
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "res")
        mp.spawn(_worker, args=(_free_port(), batches, cap, dim, where, path), nprocs=WORLD, join=True)
        res = {}
        for r in range(WORLD):
            res.update(dict(np.load(path + f".{r}.npz")))
    _, ref_codes = co.FifoEngine(cap, 0, WORLD).run(batches)
    for i, b in enumerate(batches):
        assert np.array_equal(res[f"codes{i}"], ref_codes[i]), i
        assert np.array_equal(res[f"rows{i}"], fo.synthetic_features(b, dim, seed=8)), i
