"""Full-size parity at the papers100M shape (111M nodes, 3.1B
CSR entries, fanout [15,10,5], batch 1024): the bench's proximity batches
sampled on the device (drop-in sample_batch and the pipeline's BatchSampler)
equal the CPU oracle's frontiers and distinct sets bit for bit, and the
device FIFO's per-batch counters on them equal the oracle's. The graph is
the bench's C3 graph (GPU continuum generator); hubs above 2048 neighbours
exercise the CTA kernel and the segmented walk's heavy-gap jumps."""
import os
import sys

import numpy as np
import pytest
import torch

from oracle import sampler_oracle as so

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def c3():
    sys.path.insert(0, ROOT)
    import bench
    from paper_2112_08541_b200.ordering import proximity_schedule_device
    cfg = bench.CONFIGS["c3"]
    dg = bench.make_graph(cfg, "continuum")
    order, _ = proximity_schedule_device(dg, cfg["S"], cfg["b"], seed=bench.RUN_SEED)
    off = dg.indptr.cpu().numpy()
    col = dg.indices.cpu().numpy()
    yield bench, cfg, dg, order.cpu().numpy(), off, col
    del dg
    torch.cuda.empty_cache()


def test_c3_batches_match_oracle(c3):
    bench, cfg, dg, order, off, col = c3
    import paper_2112_08541_b200 as bgl
    assert dg.num_edges > 3_000_000_000 and int(np.diff(off).max()) > 2048
    scfg = bgl.SamplingConfig(fanouts=cfg["fanouts"], seed=bench.RUN_SEED)
    b = cfg["b"]
    for i in (0, 57):
        seeds = order[i * b:(i + 1) * b].astype(np.int64)
        fr, d = bgl.sample_batch(dg, seeds, scfg, batch_seed=i)
        fr_o, _, d_o, _ = so.sample_batch(off, col, seeds, cfg["fanouts"], bench.RUN_SEED, i)
        for h, (a, e) in enumerate(zip(fr, fr_o)):
            assert np.array_equal(a, e), (i, h)
        assert np.array_equal(d, d_o), i


def test_c3_pipeline_sampler_distinct_matches_oracle(c3):
    """The pipeline's configuration of the sampler (no frontier stores, only
    dedup marks: frontier_outputs=False) gives the same distinct sets."""
    bench, cfg, dg, order, off, col = c3
    from paper_2112_08541_b200.sampler import BatchSampler, pcg_states, pcg_tables
    b = cfg["b"]
    batches = (3, 120)
    s = BatchSampler(dg, cfg["fanouts"], b, frontier_outputs=False)
    tables = pcg_tables(pcg_states(bench.RUN_SEED, range(max(batches) + 1)))
    for i in batches:
        seeds = order[i * b:(i + 1) * b]
        s.load_seeds(torch.from_numpy(seeds.astype(np.int32)).cuda())
        s.run(tables[i])
        u = int(s.num_uniq.item())
        _, _, d_o, _ = so.sample_batch(off, col, seeds.astype(np.int64), cfg["fanouts"], bench.RUN_SEED, i)
        assert np.array_equal(s.uniq[:u].cpu().numpy(), d_o), i


@pytest.mark.parametrize("d,cap,host", [(1, 1_000_000, 0), (8, 150_000, 500_000)])
def test_c3_fifo_counters_match_oracle(c3, d, cap, host):
    """FIFO cache at the papers100M shape (rings wrap, d = 8 shards with peer
    hits, the shared host level) vs the batch-parallel oracle, per batch."""
    bench, cfg, dg, order, off, col = c3
    import paper_2112_08541_b200 as bgl
    from oracle import cache_oracle as co
    from paper_2112_08541_b200.sampler import AccessTrace, BatchSampler, pcg_states, pcg_tables
    b, nb = cfg["b"], 16
    s = BatchSampler(dg, cfg["fanouts"], b, frontier_outputs=False)
    tables = pcg_tables(pcg_states(bench.RUN_SEED, range(nb)))
    batches = []
    for i in range(nb):
        s.load_seeds(torch.from_numpy(order[i * b:(i + 1) * b].astype(np.int32)).cuda())
        s.run(tables[i])
        batches.append(s.distinct().cpu().numpy().astype(np.int64))
    rep = bgl.simulate(AccessTrace(batches=batches), bgl.CacheConfig(device_capacity=cap, host_capacity=host,
                                                                     num_devices=d, feature_bytes_per_node=512))
    want, _, _ = co.simulate_batched(batches, cap, host, d)
    got = np.stack([rep.batch_queries, rep.batch_own_hits, rep.batch_peer_hits, rep.batch_host_hits,
                    rep.batch_misses, rep.batch_insertions, rep.batch_evictions], axis=1)
    assert np.array_equal(got, want)
    assert want[:, 6].sum() > 0                 # the rings wrapped


def test_c3_simulate_epoch_comm_report_matches_oracle(c3):
    """simulate_epoch with an 8-way random partition at the papers100M shape:
    trace rows and the EpochCommReport (local/remote accesses, seed and
    request loads, parent_idx-propagated origins) vs the oracle."""
    bench, cfg, dg, order, off, col = c3
    import paper_2112_08541_b200 as bgl
    b, k = cfg["b"], 8

    class P:
        pass

    p = P()
    p.part_of = np.random.default_rng(5).integers(0, k, dg.num_nodes).astype(np.int64)
    p.k = k
    batches = [order[i * b:(i + 1) * b].astype(np.int64) for i in range(3)]
    sched = bgl.BatchSchedule(batches=batches, batch_size=b, policy="proximity-S4")
    trace, rep = bgl.simulate_epoch(dg, p, sched, bgl.SamplingConfig(fanouts=cfg["fanouts"], seed=bench.RUN_SEED))
    tr_o, local, remote, seed_load, request_load = so.simulate_epoch(off, col, p.part_of, k, batches, cfg["fanouts"],
                                                                     bench.RUN_SEED)
    assert all(np.array_equal(a, e) for a, e in zip(trace.batches, tr_o))
    assert (rep.local_accesses, rep.remote_accesses) == (local, remote)
    assert np.array_equal(rep.seed_load, seed_load) and np.array_equal(rep.request_load, request_load)
