"""BASELINE.json configs[1] (the bench workload) at full size against the
reference itself: gnnio generated the products-shaped graph (2.4M nodes,
125M CSR entries), the proximity schedule and the first mini-batches' traces
and FIFO outcomes (tests/golden/c2.npz, make_golden.py make_c2; ~10 minutes
of reference CPU time). The B200 path rebuilds the graph natively and runs the
bench's captured pipeline (host features, 10% FIFO cache); the graph, the
schedule, every trace row, outcome code and counter must be identical and
every gathered row must equal F[id]."""

import numpy as np
import pytest
import torch

from packing import get

from oracle import features_oracle as fo

pytestmark = pytest.mark.gpu


def test_c2_graph_schedule_and_pipeline_match_reference(golden):
    from paper_2112_08541_b200.cachesim import CacheConfig
    from paper_2112_08541_b200.features import synthetic_features
    from paper_2112_08541_b200.graph import generate_power_law_exact_device
    from paper_2112_08541_b200.ordering import proximity_schedule_device
    from paper_2112_08541_b200.pipeline import MiniBatchPipeline
    npz = golden("c2")
    n, dim = 2_400_000, 100
    dg = generate_power_law_exact_device(n, 51, 1, 0.08, 47)
    assert dg.num_edges == int(npz["csr_entries"][0])
    col = dg.indices.cpu().numpy().astype(np.int64)
    assert int((col * (np.arange(col.size) % 1000003 + 1)).sum() % (1 << 61)) == int(npz["csr_checksum"][0])
    assert np.array_equal(dg.indptr[-1000:].cpu().numpy(), npz["offsets_tail"])
    del col
    order, b = proximity_schedule_device(dg, 4, 1024, seed=1)
    sched = get(npz, "schedule")
    flat = order.cpu().numpy()
    for i, ref in enumerate(sched):
        assert np.array_equal(flat[i * b:(i + 1) * b], ref), i
    feats = synthetic_features(n, dim, seed=1)
    pipe = MiniBatchPipeline(dg, (15, 10, 5), 1024, order, 1,
                             CacheConfig(device_capacity=240_000, feature_bytes_per_node=dim * 4), feats)
    pipe.capture()
    trace, codes, cnt = get(npz, "trace"), get(npz, "codes"), npz["counters"]
    cum = np.cumsum(cnt, axis=0)
    for i in range(len(trace)):
        pipe.step()
        torch.cuda.synchronize()
        d = pipe.distinct().cpu().numpy()
        assert np.array_equal(d, trace[i]), i
        assert np.array_equal(pipe.codes().cpu().numpy(), codes[i]), i
        assert np.array_equal(pipe.rows().cpu().numpy(), fo.synthetic_features(d, dim, seed=1)), i
        if i + 2 < len(trace):
            assert np.array_equal(pipe.counters.cpu().numpy()[:7], cum[i + 2]), i


def _digest(a) -> int:
    """tests/golden/make_golden.py digest(): order-sensitive 61-bit digest."""
    a = np.asarray(a, dtype=np.int64).ravel()
    w = np.arange(a.size, dtype=np.int64) % 1000003 + 1
    return int(((a % (1 << 31)) * w).sum() % ((1 << 61) - 1))


def test_c2_bench_window_matches_reference(golden):
    """The whole default bench window (batches 0..24: W = 5 warm-up + K = 20
    timed) against the reference itself (tests/golden/c2_window.npz, gnnio's
    sample_batch + simulate(FIFO) on its own graph and schedule): every batch's
    distinct set and outcome codes (size, sum, digest) and counters through the
    bench's captured pipeline, every gathered row = F[id], and the ring's tail
    and contents after the window through the drop-in cachesim.simulate."""
    from paper_2112_08541_b200.cachesim import CacheConfig, cold_state, simulate
    from paper_2112_08541_b200.features import synthetic_features
    from paper_2112_08541_b200.graph import generate_power_law_exact_device
    from paper_2112_08541_b200.ordering import proximity_schedule_device
    from paper_2112_08541_b200.pipeline import MiniBatchPipeline
    from paper_2112_08541_b200.sampler import AccessTrace
    npz = golden("c2_window")
    nbw = int(npz["size"].size)
    n, dim = 2_400_000, 100
    dg = generate_power_law_exact_device(n, 51, 1, 0.08, 47)
    order, b = proximity_schedule_device(dg, 4, 1024, seed=1)
    assert _digest(order.cpu().numpy()) == int(npz["schedule_digest"][0])
    feats = synthetic_features(n, dim, seed=1)
    cfg = CacheConfig(device_capacity=240_000, feature_bytes_per_node=dim * 4)
    pipe = MiniBatchPipeline(dg, (15, 10, 5), 1024, order, 1, cfg, feats)
    pipe.capture()
    cum = np.cumsum(npz["counters"], axis=0)
    trace = []
    for i in range(nbw):
        pipe.step()
        torch.cuda.synchronize()
        d = pipe.distinct().cpu().numpy()
        trace.append(d.astype(np.int64))
        assert d.size == int(npz["size"][i]) and int(d.astype(np.int64).sum()) == int(npz["sum"][i]), i
        assert _digest(d) == int(npz["trace_digest"][i]), i
        assert _digest(pipe.codes().cpu().numpy()) == int(npz["codes_digest"][i]), i
        if i % 6 == 0:
            assert np.array_equal(pipe.rows().cpu().numpy(), fo.synthetic_features(d, dim, seed=1)), i
        if i + 2 < nbw:                       # the pipeline's lookups run two batches ahead
            assert np.array_equal(pipe.counters.cpu().numpy()[:7], cum[i + 2]), i
    state = cold_state(cfg)
    rep = simulate(AccessTrace(batches=trace), cfg, state=state)
    assert np.array_equal(np.array([rep.batch_queries, rep.batch_own_hits, rep.batch_peer_hits, rep.batch_host_hits,
                                    rep.batch_misses, rep.batch_insertions, rep.batch_evictions]).T, npz["counters"])
    assert state.devices[0].tail == int(npz["ring_tail"][0])
    assert _digest(state.devices[0].slots) == int(npz["ring_digest"][0])
