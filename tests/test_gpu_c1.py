"""BASELINE.json configs[0] (C1) end to end against the reference itself:
gnnio generated the graph, the proximity schedule, the epoch's access trace
and the FIFO cache outcomes (tests/golden/c1.npz, make_golden.py make_c1).
Here the B200 path rebuilds the same graph (native generator), schedules on
the device, and runs the drop-in API (simulate_epoch + simulate) and the
captured 5-branch pipeline over the whole epoch; every schedule entry, trace
row, outcome code and per-batch counter must be identical, and every gathered
row must equal F[id]."""

import numpy as np
import pytest
import torch

from packing import get

from oracle import features_oracle as fo

pytestmark = pytest.mark.gpu

N, AVG, SEED, TRAIN, LABELS, S, B, FAN, CAP, DIM = 100_000, 20, 1, 0.1, 64, 4, 1024, (10, 5), 10_000, 128


@pytest.fixture(scope="module")
def c1(golden):
    from paper_2112_08541_b200.graph import generate_power_law_exact_device
    npz = golden("c1")
    dg = generate_power_law_exact_device(N, AVG, SEED, TRAIN, LABELS)
    assert dg.num_edges == int(npz["csr_entries"][0])
    return npz, dg


def test_c1_schedule_trace_and_cache_through_the_drop_in_api(c1):
    import paper_2112_08541_b200 as bgl
    npz, dg = c1
    sched = bgl.proximity_schedule(dg, S, B, seed=SEED)
    ref_sched = get(npz, "schedule")
    assert len(sched.batches) == len(ref_sched)
    assert all(np.array_equal(a, b) for a, b in zip(sched.batches, ref_sched))

    class OnePartition:            # random_partition(g, 1): every node in partition 0
        k = 1
        part_of = np.zeros(N, dtype=np.int64)

    trace, _ = bgl.simulate_epoch(dg, OnePartition(), sched, bgl.SamplingConfig(fanouts=FAN, batch_size=B, seed=SEED))
    ref_trace = get(npz, "trace")
    assert all(np.array_equal(a, b) for a, b in zip(trace.batches, ref_trace))
    rep = bgl.simulate(trace, bgl.CacheConfig(device_capacity=CAP, policy="fifo", feature_bytes_per_node=DIM * 4),
                       record_outcomes=True)
    got = np.array([rep.batch_queries, rep.batch_own_hits, rep.batch_peer_hits, rep.batch_host_hits,
                    rep.batch_misses, rep.batch_insertions, rep.batch_evictions]).T
    assert np.array_equal(got, npz["counters"])
    assert rep.outcomes == [["DPHM"[c] for c in cd] for cd in get(npz, "codes")]


@pytest.mark.parametrize("where", ["host", "hbm"])
def test_c1_pipeline_epoch_matches_reference(c1, where):
    from paper_2112_08541_b200.cachesim import CacheConfig
    from paper_2112_08541_b200.features import synthetic_features
    from paper_2112_08541_b200.ordering import proximity_schedule_device
    from paper_2112_08541_b200.pipeline import MiniBatchPipeline
    npz, dg = c1
    order, _ = proximity_schedule_device(dg, S, B, seed=SEED)
    feats = synthetic_features(N, DIM, seed=3, device_resident=(where == "hbm"))
    pipe = MiniBatchPipeline(dg, FAN, B, order, SEED, CacheConfig(device_capacity=CAP, feature_bytes_per_node=DIM * 4),
                             feats)
    pipe.capture()
    trace, codes, cnt = get(npz, "trace"), get(npz, "codes"), npz["counters"]
    cum = np.cumsum(cnt, axis=0)
    nb = len(trace)
    for i in range(nb):
        pipe.step()
        torch.cuda.synchronize()
        d = pipe.distinct().cpu().numpy()
        assert np.array_equal(d, trace[i]), i
        assert np.array_equal(pipe.codes().cpu().numpy(), codes[i]), i
        assert np.array_equal(pipe.rows().cpu().numpy(), fo.synthetic_features(d, DIM, seed=3)), i
        if i + 2 < nb:             # LI(i+2) ran in step i
            assert np.array_equal(pipe.counters.cpu().numpy()[:7], cum[i + 2]), i
