"""World-size-2 CPU (gloo) test of the multi-GPU exchange protocol of the
node-ID-sharded cache (paper_2112_08541_b200/distributed.py).

The per-home engine and the partition/scatter ops are replaced by the CPU
oracle (test infrastructure); the protocol itself -- bucketing by home, ID
all-to-all, worker-ordered serving at every home, row/code all-to-all back,
scatter into batch order -- is the product code. Result must equal the
reference's single-process d-device simulation: per-node codes D/P/M and
rows F[batch]."""

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

DIM = 8
WORLD = 2


class CpuOps:
    def partition(self, ids):
        home = ids % WORLD
        order = torch.argsort(home, stable=True)
        counts = torch.bincount(home.long(), minlength=WORLD).to(torch.int64)
        return ids[order], order.to(torch.int32), counts

    def scatter(self, pos, rows, out):
        out[pos.long()] = rows


class OracleShard:
    """Home shard `rank`: oracle FIFO ring + synthetic feature table."""

    def __init__(self, rank, cap):
        self.rank = rank
        self.ring = co.FifoRing(cap)
        self.counters = torch.zeros(8, dtype=torch.int64)

    def serve(self, ids, worker, rows_out, codes_out):
        v = ids.numpy()
        codes = np.array([(co.CODE_D if worker == self.rank else co.CODE_P) if int(x) in self.ring else co.CODE_M
                          for x in v], dtype=np.uint8)
        for x in sorted(int(x) for x, c in zip(v, codes) if c == co.CODE_M):
            self.ring.insert(x)
        codes_out[:] = torch.from_numpy(codes)
        rows_out[:] = torch.from_numpy(fo.synthetic_features(v, DIM, seed=4))


def _worker(rank, port, batches, cap, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_2112_08541_b200.distributed import ShardedFeatureCache
    sc = ShardedFeatureCache(rank, WORLD, OracleShard(rank, cap), CpuOps(), DIM, device=torch.device("cpu"))
    out = {}
    for j in range(len(batches) // WORLD):
        i = j * WORLD + rank
        rows, codes = sc.step(torch.from_numpy(batches[i].astype(np.int32)))
        out[f"rows{i}"] = rows.numpy()
        out[f"codes{i}"] = codes.numpy()
    np.savez(path + f".{rank}.npz", **out)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("cap", [3, 40])
def test_sharded_exchange_matches_reference_simulation(cap):
    rng = np.random.default_rng(5)
    batches = [np.unique(rng.integers(0, 120, size=int(rng.integers(5, 40)))) for _ in range(12)]
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "res")
        mp.spawn(_worker, args=(_free_port(), batches, cap, path), nprocs=WORLD, join=True)
        res = {}
        for r in range(WORLD):
            res.update(dict(np.load(path + f".{r}.npz")))
    # reference semantics: d = WORLD device levels, worker of batch i = i % d
    _, ref_codes = co.FifoEngine(cap, 0, WORLD).run(batches)
    for i, b in enumerate(batches):
        assert np.array_equal(res[f"codes{i}"], ref_codes[i]), i
        assert np.array_equal(res[f"rows{i}"], fo.synthetic_features(b, DIM, seed=4)), i
