"""GPU test of the pipelined, host-sync-free sharded round (ShardedPipeline):
two (or three) processes share one GPU (CUDA IPC works between processes of
one device), each is home shard `rank` and worker of every world-th batch.
IDs reach the homes through bgl_partition_push (peer stores), codes and hit
rows come back through the homes' pushes, each worker fetches its own misses;
a host barrier stands in for the NCCL one (NCCL cannot put two ranks on one
GPU). Every round's distinct set, per-node outcome codes and rows must equal
the reference: the oracle sampler + the reference's d-device FIFO simulation
(cachesim.py:275-363) + F[ids]."""

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
from oracle import sampler_oracle as so

pytestmark = pytest.mark.gpu
WORLD = 2
N, DEG, FAN, B, SEED, DIM = 20000, 10, (10, 5), 256, 6, 32


def _graph():
    from paper_2112_08541_b200.graph import generate_power_law_exact_device
    return generate_power_law_exact_device(N, DEG, seed=3, train_fraction=0.2, num_labels=4)


def _order():
    dg_train = np.arange(N)[np.random.default_rng(1).permutation(N)][: 24 * B]
    return dg_train.astype(np.int32)


def _route(world, rounds):
    """batch_devices with a different permutation of the GPUs every round."""
    rng = np.random.default_rng(world * 7 + rounds)
    return [int(w) for _ in range(rounds) for w in rng.permutation(world)]


def _worker(rank, world, port, cap, where, rounds, path, host=0, routed=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2112_08541_b200.distributed import ShardedPipeline
    from paper_2112_08541_b200.features import synthetic_features

    def host_barrier():
        torch.cuda.synchronize()
        dist.barrier()

    dg = _graph()
    feats = synthetic_features(N, DIM, seed=8, device_resident=(where == "hbm"))
    order = torch.from_numpy(_order()).cuda()
    pipe = ShardedPipeline(rank, world, dg, FAN, B, order, SEED, cap, feats, num_batches=rounds * world,
                           barrier=host_barrier, host_capacity=host,
                           batch_devices=_route(world, rounds) if routed else None)
    out = {}
    for j in range(rounds):
        pipe.step()
        torch.cuda.synchronize()
        i = pipe.batch_of(j)
        out[f"ids{i}"] = pipe.distinct(j).cpu().numpy()
        out[f"rows{i}"] = pipe.rows(j).cpu().numpy()
        out[f"codes{i}"] = pipe.outcome_codes(j).cpu().numpy()
        host_barrier()            # nobody starts round j+2 (overwriting parity j) before all have read j
    out["counters"] = pipe.counters.cpu().numpy()
    np.savez(path + f".{rank}.npz", **out)
    dist.barrier()
    pipe.close()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("where,cap,world,host,routed", [("host", 700, 2, 0, False), ("hbm", 300, 2, 0, False),
                                                         ("host", 500, 3, 0, False), ("host", 600, 2, 8, False),
                                                         ("host", 400, 3, 64, False), ("host", 500, 2, 0, True),
                                                         ("hbm", 300, 3, 64, True)])
def test_sharded_pipeline_matches_reference(where, cap, world, host, routed):
    """... with the shared host level on GPU 0 (host = its capacity,
    cachesim.py:202, 330-344) and with batch_devices routing (a different GPU
    permutation every round, cachesim.py:309) against the reference's
    d-device simulation with the same host level and routing."""
    rounds = 6
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "res")
        mp.spawn(_worker, args=(world, _free_port(), cap, where, rounds, path, host, routed), nprocs=world,
                 join=True)
        res = {}
        for r in range(world):
            res.update({k + (f"_r{r}" if k == "counters" else ""): v for k, v in np.load(path + f".{r}.npz").items()})
    # reference: same graph on the host, oracle sampler, 2-device FIFO simulation
    from paper_2112_08541_b200.graph import power_law_edges
    from oracle import graph_oracle as go
    edges, _, _ = power_law_edges(N, DEG, 3, 0.2, 4)
    off, col = go.csr_from_edges(edges.astype(np.int64), N)
    order = _order()
    nb = rounds * world
    distinct = [so.sample_batch(off, col, order[i * B:(i + 1) * B].astype(np.int64), FAN, SEED, i)[2]
                for i in range(nb)]
    # the pipeline's lookups run two rounds ahead (LI(k+2) in step k): rounds
    # 0..rounds+1, batch indices wrapping over the epoch
    seq = [distinct[i % nb] for i in range((rounds + 2) * world)]
    route = _route(world, rounds) if routed else None
    bd = None if route is None else [route[i % nb] for i in range(len(seq))]
    eng = co.FifoEngine(cap, host, world)
    ref_cnt, ref_codes = eng.run(seq, bd)
    for i in range(nb):
        assert np.array_equal(res[f"ids{i}"], distinct[i]), i
        assert np.array_equal(res[f"codes{i}"], ref_codes[i]), i
        assert np.array_equal(res[f"rows{i}"], fo.synthetic_features(distinct[i], DIM, seed=8)), i
    tot = sum(res[f"counters_r{r}"] for r in range(world))
    ref = np.asarray(ref_cnt).sum(axis=0)
    if host == 0:
        assert tot[:7].tolist() == ref[:7].tolist()
        return
    # the device levels' lookups ran two rounds ahead, the host level (step k
    # serves round k) did not: H, host inserts and evictions cover rounds 0..R-1
    first = co.FifoEngine(cap, host, world)
    cnt_r, _ = first.run(seq[:nb], None if bd is None else bd[:nb])
    h_r = int(np.asarray(cnt_r)[:, 3].sum())
    assert tot[:3].tolist() == ref[:3].tolist()
    assert int(tot[3]) == h_r and int(tot[3] + tot[4]) == int(ref[3] + ref[4])
    assert int(tot[5]) == int(ref[5]) - eng.host.insertions + first.host.insertions
    assert int(tot[6]) == int(ref[6]) - eng.host.evictions + first.host.evictions


def test_sharded_pipeline_graphs_single_rank_nccl():
    """World size 1 over NCCL: the captured step (12 phases, NCCL barrier
    inside) replays the same rounds as the eager steps, and both equal the
    reference's 1-device FIFO simulation + F[ids]."""
    import torch.distributed as dist
    from paper_2112_08541_b200.distributed import ShardedPipeline
    from paper_2112_08541_b200.features import synthetic_features
    from paper_2112_08541_b200.graph import power_law_edges
    from oracle import graph_oracle as go
    if dist.is_initialized():
        pytest.skip("process group already initialised")
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        dg = _graph()
        feats = synthetic_features(N, DIM, seed=8)
        order = torch.from_numpy(_order()).cuda()
        nb, cap = 12, 500
        pipe = ShardedPipeline(0, 1, dg, FAN, B, order, SEED, cap, feats, num_batches=nb)
        got = {}
        for j in range(30):
            if j == 3:
                pipe.capture()
            pipe.step()
            torch.cuda.synchronize()
            got[j] = (pipe.distinct(j).cpu().numpy(), pipe.outcome_codes(j).cpu().numpy(),
                      pipe.rows(j).cpu().numpy())
        pipe.close()
    finally:
        dist.destroy_process_group()
    edges, _, _ = power_law_edges(N, DEG, 3, 0.2, 4)
    off, col = go.csr_from_edges(edges.astype(np.int64), N)
    order_h = _order()
    distinct = [so.sample_batch(off, col, order_h[i * B:(i + 1) * B].astype(np.int64), FAN, SEED, i)[2]
                for i in range(nb)]
    _, ref_codes = co.FifoEngine(cap, 0, 1).run([distinct[j % nb] for j in range(30)])
    for j in range(30):
        ids, codes, rows = got[j]
        assert np.array_equal(ids, distinct[j % nb]), j
        assert np.array_equal(codes, ref_codes[j]), j
        assert np.array_equal(rows, fo.synthetic_features(ids, DIM, seed=8)), j


def _shm_worker(rank, port, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_2112_08541_b200.features import shared_synthetic_features, table_pointer
    from paper_2112_08541_b200 import _lib
    n, dim = 50000, 24
    t, plan = shared_synthetic_features(n, dim, 5, f"bgl_test_{port}", rank, WORLD, dist.barrier, chunk_rows=7000)
    ids = torch.from_numpy(np.random.default_rng(rank).integers(0, n, 3000).astype(np.int32)).cuda()
    pos = torch.arange(3000, dtype=torch.int32, device="cuda")
    cnt = torch.tensor([3000], dtype=torch.int64, device="cuda")
    out = torch.empty((3000, dim), dtype=torch.float32, device="cuda")
    _lib.call("bgl_gather_list", pos.data_ptr(), cnt.data_ptr(), 3000, ids.data_ptr(), table_pointer(t), dim * 4,
              out.data_ptr(), None, None, 2, 16, _lib.stream_ptr())
    torch.cuda.synchronize()
    np.savez(path + f".{rank}.npz", ids=ids.cpu().numpy(), rows=out.cpu().numpy(), host=t[::997].numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_shared_feature_store_across_processes():
    """The /dev/shm feature store filled cooperatively by two processes and
    registered by both: zero-copy gathers read F[ids] in each process."""
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "shm")
        port = _free_port()
        mp.spawn(_shm_worker, args=(port, path), nprocs=WORLD, join=True)
        for r in range(WORLD):
            z = np.load(path + f".{r}.npz")
            assert np.array_equal(z["rows"], fo.synthetic_features(z["ids"], 24, seed=5))
            assert np.array_equal(z["host"], fo.synthetic_features(np.arange(0, 50000, 997), 24, seed=5))
        assert not os.path.exists(f"/dev/shm/bgl_test_{port}")
