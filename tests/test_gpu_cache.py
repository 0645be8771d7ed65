"""GPU parity: FIFO cache engine and feature gather vs the reference's golden
vectors and the CPU oracle (bit-exact)."""

import numpy as np
import pytest
import torch

from packing import get

from oracle import cache_oracle as co
from oracle import features_oracle as fo

pytestmark = pytest.mark.gpu


def _cases(npz):
    specs = npz["specs"]
    batches = get(npz, "batches")
    codes = get(npz, "codes")
    dsl = get(npz, "dev_slots")
    dtl = get(npz, "dev_tails")
    hsl = get(npz, "host_slots")
    htl = get(npz, "host_tails")
    cnt = npz["counters"]
    b0 = 0
    for ci, (d, cap, hcap, nb, use_bd, kind) in enumerate(specs):
        bd = npz[f"bd_{ci}"].tolist() if use_bd else None
        sl = slice(b0, b0 + nb)
        yield ci, int(d), int(cap), int(hcap), bd, batches[sl], codes[sl], cnt[sl], dsl[sl], dtl[sl], hsl[sl], htl[ci]
        b0 += nb


def test_fifo_whole_trace_matches_reference(golden):
    from paper_2112_08541_b200 import cachesim as cs
    from paper_2112_08541_b200.sampler import AccessTrace
    npz = golden("cache")
    for ci, d, cap, hcap, bd, batches, codes, cnt, dsl, dtl, hsl, htl in _cases(npz):
        cfg = cs.CacheConfig(device_capacity=cap, host_capacity=hcap, num_devices=d, feature_bytes_per_node=400)
        rep = cs.simulate(AccessTrace(batches=batches), cfg, batch_devices=bd, record_outcomes=True)
        assert np.array_equal(np.array([rep.batch_queries, rep.batch_own_hits, rep.batch_peer_hits,
                                        rep.batch_host_hits, rep.batch_misses, rep.batch_insertions,
                                        rep.batch_evictions, rep.batch_metadata_updates]).T, cnt), ci
        assert rep.outcomes == [["DPHM"[c] for c in cd] for cd in codes], ci


def test_fifo_eviction_order_every_batch(golden):
    """Ring contents + tail of every level after every batch (state= path)."""
    from paper_2112_08541_b200 import cachesim as cs
    from paper_2112_08541_b200.sampler import AccessTrace
    npz = golden("cache")
    for ci, d, cap, hcap, bd, batches, codes, cnt, dsl, dtl, hsl, htl in _cases(npz):
        if ci % 3:
            continue
        cfg = cs.CacheConfig(device_capacity=cap, host_capacity=hcap, num_devices=d)
        state = cs.cold_state(cfg)
        for i, b in enumerate(batches):
            cs.simulate(AccessTrace(batches=[b]), cfg, batch_devices=[bd[i] if bd else i % d], state=state)
            ds, dt, hs, ht = state.engine.export()
            assert np.array_equal(ds.ravel(), dsl[i]), (ci, i)
            assert dt.tolist() == dtl[i].tolist()
            assert np.array_equal(hs, hsl[i])
            assert ht == htl[i]
        assert len(state.devices[0]) <= cap


def test_fifo_real_trace(golden):
    from paper_2112_08541_b200 import cachesim as cs
    from paper_2112_08541_b200.sampler import AccessTrace
    npz = golden("cache")
    trace = AccessTrace(batches=get(npz, "real_trace"))
    for j, d in enumerate((1, 2, 4, 8)):
        rep = cs.simulate(trace, cs.CacheConfig(device_capacity=500 // d, host_capacity=250, num_devices=d))
        got = np.array([rep.batch_queries, rep.batch_own_hits, rep.batch_peer_hits, rep.batch_host_hits,
                        rep.batch_misses, rep.batch_insertions, rep.batch_evictions])
        assert np.array_equal(got, npz["real_counters"][j])


def test_reference_hand_cases():
    from paper_2112_08541_b200 import cachesim as cs
    from paper_2112_08541_b200.sampler import AccessTrace

    def tr(*b):
        return AccessTrace(batches=[np.array(x, dtype=np.int64) for x in b])

    rep = cs.simulate(tr([0, 1], [2], [0]), cs.CacheConfig(device_capacity=2))
    assert rep.batch_misses == [2, 1, 1] and rep.hit_ratio == 0.0
    rep = cs.simulate(tr([3], [3]), cs.CacheConfig(device_capacity=4, num_devices=2), batch_devices=[0, 0],
                      record_outcomes=True)
    assert rep.outcomes == [["M"], ["P"]]
    rep = cs.simulate(tr([0, 1], [0, 1], [0, 1]), cs.CacheConfig(device_capacity=1, host_capacity=8),
                      record_outcomes=True)
    assert rep.outcomes[0] == ["M", "M"] and rep.misses == 2
    rep = cs.simulate(tr([0, 1], [2, 0]), cs.CacheConfig(device_capacity=0))
    assert rep.hit_ratio == 0.0 and rep.misses == 4
    with pytest.raises(ValueError, match="mismatch"):
        st = cs.cold_state(cs.CacheConfig(device_capacity=2))
        st.policy = "lru"
        cs.simulate(tr([0]), cs.CacheConfig(device_capacity=2), state=st)
    # LRU / LFU run on the device too (tests/test_gpu_ordered.py); FeatureCacheEngine stays FIFO
    rep = cs.simulate(tr([0], [0]), cs.CacheConfig(device_capacity=2, policy="lru"), record_outcomes=True)
    assert rep.outcomes == [["M"], ["D"]] and rep.batch_metadata_updates == [1, 1]


@pytest.mark.parametrize("where", ["host", "hbm"])
@pytest.mark.parametrize("d", [1, 4])
def test_feature_retrieval_bit_exact(where, d):
    from paper_2112_08541_b200 import cachesim as cs
    from paper_2112_08541_b200.features import FeatureCacheEngine, synthetic_features
    n, dim = 20000, 100
    feats = synthetic_features(n, dim, seed=9, device_resident=(where == "hbm"))
    ref_table = fo.synthetic_features(np.arange(n), dim, seed=9)
    assert np.array_equal(feats.cpu().numpy(), ref_table)
    rng = np.random.default_rng(3)
    batches = [np.unique(rng.integers(0, 3000 + 1000 * i, size=2500)) for i in range(12)]
    cfg = cs.CacheConfig(device_capacity=1500 // d, host_capacity=0, num_devices=d, feature_bytes_per_node=400)
    eng = FeatureCacheEngine(cfg, feats, max_batch=max(len(b) for b in batches))
    oracle = co.FifoEngine(cfg.device_capacity, 0, d)
    for i, b in enumerate(batches):
        rows, codes = eng.retrieve(b, i)
        assert np.array_equal(rows.cpu().numpy(), ref_table[b]), i
        _, ocodes = oracle.run([b], [i % d])
        assert np.array_equal(codes.cpu().numpy(), ocodes[0]), i
    # the ring rows hold exactly the features of the resident nodes
    from paper_2112_08541_b200 import _lib
    ds, _, _, _ = eng.dev.export()
    flat = ds.ravel()
    slots = np.flatnonzero(flat >= 0)
    src = torch.from_numpy(slots.astype(np.int64)).cuda()
    ids = torch.from_numpy(flat[slots].astype(np.int32)).cuda()
    nd = torch.tensor([len(slots)], dtype=torch.int64, device="cuda")
    out = torch.empty((len(slots), dim), dtype=torch.float32, device="cuda")
    _lib.call("bgl_gather_rows", ids.data_ptr(), src.data_ptr(), nd.data_ptr(), len(slots), eng.dev.rows_ptr(),
              eng.table, dim * 4, out.data_ptr(), 0, 0, _lib.stream_ptr())
    assert np.array_equal(out.cpu().numpy(), ref_table[flat[slots]])


def test_static_degree_policy_matches_reference(golden):
    from conftest import golden_graph
    from test_oracle_golden import _static_cases

    from paper_2112_08541_b200 import cachesim as cs
    from paper_2112_08541_b200.sampler import AccessTrace

    class G:
        def __init__(self, off, col):
            self.row_offsets, self.col_indices, self.num_nodes = off, col, len(off) - 1

    npz = golden("static")
    for gname, d, cap, hcap, dsets, hset, batches, codes, cnt in _static_cases(npz):
        off, col, _ = golden_graph(npz, gname)
        g = G(off, col)
        cfg = cs.CacheConfig(device_capacity=cap, host_capacity=hcap, num_devices=d, policy="static-degree")
        state = cs.warm_static(g, cfg)
        assert [sorted(lv.resident) for lv in state.devices] == [x.tolist() for x in dsets], (gname, d, cap)
        assert sorted(state.host.resident) == hset.tolist()
        rep = cs.simulate(AccessTrace(batches=batches), cfg, g=g, record_outcomes=True)
        got = np.array([rep.batch_queries, rep.batch_own_hits, rep.batch_peer_hits, rep.batch_host_hits,
                        rep.batch_misses, rep.batch_insertions, rep.batch_evictions]).T
        assert np.array_equal(got, cnt)
        assert rep.outcomes == [["DPHM"[c] for c in cd] for cd in codes]
        assert sum(rep.batch_metadata_updates) == 0
    with pytest.raises(ValueError):
        cs.cold_state(cs.CacheConfig(device_capacity=2, policy="static-degree"))


@pytest.mark.parametrize("rows_in_flight", [2, 4, 8])
@pytest.mark.parametrize("where", ["host", "hbm"])
def test_compacted_miss_list_and_gather(rows_in_flight, where):
    """bgl_cache_lookup_misses writes exactly the ascending positions of the
    device misses; bgl_gather_list fills those rows (and only those) with
    F[id], plus the home-push copy at push_pos; the hit rows come from the
    ring after the insert. Three batches through one engine vs the oracle."""
    from paper_2112_08541_b200 import _lib
    from paper_2112_08541_b200.cachesim import CacheConfig
    from paper_2112_08541_b200.features import FeatureCacheEngine, synthetic_features

    rng = np.random.default_rng(7)
    n, dim, cap = 50000, 100, 3000
    feats = synthetic_features(n, dim, seed=3, device_resident=(where == "hbm"))
    eng = FeatureCacheEngine(CacheConfig(device_capacity=cap, feature_bytes_per_node=dim * 4), feats, max_batch=8000)
    fifo = co.FifoEngine(cap, 0, 1)
    lib = _lib.load()
    for bi in range(3):
        ids_np = np.unique(rng.integers(0, n // 4 if bi else n, 6000))
        _, ref_codes = fifo.run([ids_np], [0])
        ids = torch.from_numpy(ids_np.astype(np.int32)).cuda()
        m = len(ids_np)
        eng.n_dev.fill_(m)
        codes = torch.empty(m, dtype=torch.uint8, device="cuda")
        src = torch.empty(m, dtype=torch.int64, device="cuda")
        mpos = torch.full((m,), -7, dtype=torch.int32, device="cuda")
        mcnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
        out = torch.zeros((m, dim), dtype=torch.float32, device="cuda")
        push = torch.zeros((m + 5, dim), dtype=torch.float32, device="cuda")
        push_pos = torch.from_numpy(rng.permutation(m + 5)[:m].astype(np.int32)).cuda()
        _lib.check(lib.bgl_cache_lookup_misses(eng.dev.handle, ids.data_ptr(), eng.n_dev.data_ptr(), m, 0,
                                               codes.data_ptr(), src.data_ptr(), cnt.data_ptr(), mpos.data_ptr(),
                                               mcnt.data_ptr(), _lib.stream_ptr()))
        assert np.array_equal(codes.cpu().numpy(), ref_codes[0])
        miss = np.flatnonzero(ref_codes[0] >= 2)
        assert int(mcnt.item()) == len(miss)
        assert np.array_equal(mpos[: len(miss)].cpu().numpy(), miss)
        _lib.check(lib.bgl_gather_list(mpos.data_ptr(), mcnt.data_ptr(), m, ids.data_ptr(), eng.table,
                                       eng.row_bytes, out.data_ptr(), push.data_ptr(), push_pos.data_ptr(),
                                       rows_in_flight, 0 if where == "hbm" else 37, _lib.stream_ptr()))
        torch.cuda.synchronize()
        ref = fo.synthetic_features(ids_np, dim, seed=3)
        o = out.cpu().numpy()
        assert np.array_equal(o[miss], ref[miss])
        hit = np.flatnonzero(ref_codes[0] < 2)
        assert not o[hit].any()                      # only the listed rows were written
        assert np.array_equal(push.cpu().numpy()[push_pos.cpu().numpy()[miss]], ref[miss])
        # hits from the ring, then insert-after-batch with the rows
        _lib.check(lib.bgl_gather_rows(ids.data_ptr(), src.data_ptr(), eng.n_dev.data_ptr(), m,
                                       eng.dev.rows_ptr(), eng.table, eng.row_bytes, out.data_ptr(), 1, 0,
                                       _lib.stream_ptr()))
        _lib.check(lib.bgl_cache_insert(eng.dev.handle, ids.data_ptr(), m, out.data_ptr(), cnt.data_ptr(),
                                        _lib.stream_ptr()))
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), ref)


@pytest.mark.parametrize("dim", [16, 100, 128])
@pytest.mark.parametrize("where", ["host", "hbm"])
def test_span_gather_matches_rows(dim, where):
    """bgl_gather_spans: runs of consecutive IDs (TMA bulk copies) and single
    rows (16-B loads) in a compacted miss list; exactly the listed rows are
    written, each equal to F[id]; runs cross the 16-entry chunks."""
    from paper_2112_08541_b200 import _lib
    from paper_2112_08541_b200.features import synthetic_features, table_pointer
    rng = np.random.default_rng(dim)
    n = 40000
    feats = synthetic_features(n, dim, seed=4, device_resident=(where == "hbm"))
    # a sorted distinct batch made of runs of random lengths
    starts = np.sort(rng.choice(n - 40, 900, replace=False))
    batch = np.unique(np.concatenate([np.arange(s, s + rng.integers(1, 30)) for s in starts]))
    batch = batch[batch < n]
    miss = np.sort(rng.choice(len(batch), int(0.6 * len(batch)), replace=False)).astype(np.int32)
    ids = torch.from_numpy(batch.astype(np.int32)).cuda()
    pos = torch.from_numpy(miss).cuda()
    cnt = torch.tensor([len(miss)], dtype=torch.int64, device="cuda")
    out = torch.zeros((len(batch), dim), dtype=torch.float32, device="cuda")
    _lib.call("bgl_gather_spans", pos.data_ptr(), cnt.data_ptr(), len(batch), ids.data_ptr(), table_pointer(feats),
              dim * 4, out.data_ptr(), 0 if where == "hbm" else 37, _lib.stream_ptr())
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    ref = fo.synthetic_features(batch, dim, seed=4)
    assert np.array_equal(o[miss], ref[miss])
    rest = np.setdiff1d(np.arange(len(batch)), miss)
    assert not o[rest].any()
    # empty list
    cnt.zero_()
    _lib.call("bgl_gather_spans", pos.data_ptr(), cnt.data_ptr(), len(batch), ids.data_ptr(), table_pointer(feats),
              dim * 4, out.data_ptr(), 0, _lib.stream_ptr())
    torch.cuda.synchronize()


def test_compare_policies_and_amortized_ops_match_reference(golden):
    """compare_policies with the reference's default policy set (POLICIES:
    static-degree, FIFO, LRU, LFU -- every cell on the device) and
    amortized_update_ops of the dynamic policies equal the reference's on a
    sampled trace (tests/golden/policies.npz; cachesim.py:366-409)."""
    from paper_2112_08541_b200 import cachesim as cs
    from paper_2112_08541_b200.sampler import AccessTrace
    from conftest import golden_graph
    npz = golden("policies")
    g_npz = golden("sampler")
    off, col, train = golden_graph(g_npz, "dense")

    class Gr:
        row_offsets, col_indices, num_nodes, train_mask = off, col, len(off) - 1, train

    trace = AccessTrace(batches=[b.astype(np.int64) for b in get(npz, "trace")])
    rows = cs.compare_policies(Gr(), trace, [40, 150, 600], num_devices=2, host_capacity=100)
    got = np.array([[list(cs.POLICIES).index(r["policy"]), r["capacity"], r["device_hits"], r["host_hits"],
                     r["misses"]] for r in rows])
    assert np.array_equal(got, npz["rows"])
    assert [r["hit_ratio"] for r in rows] == npz["hit_ratio"].tolist()
    for j, p in enumerate(("fifo", "lru", "lfu")):
        amort = cs.amortized_update_ops(cs.simulate(trace, cs.CacheConfig(device_capacity=150, host_capacity=100,
                                                                          num_devices=2, policy=p)))
        assert [amort[k] for k in ("lookups_per_batch", "insertions_per_batch", "evictions_per_batch",
                                   "metadata_updates_per_batch")] == npz["amortized"][j].tolist(), p


@pytest.mark.parametrize("d,cap,hcap", [(1, 40, 0), (3, 17, 8), (4, 0, 16), (2, 64, 64)])
def test_level_counters_match_reference_levels(d, cap, hcap):
    """FifoLevelView.insertions / .evictions / .metadata_updates of every
    device level and of the host level equal the reference levels' counters
    (_Level, cachesim.py:45-49; FifoLevel.insert :94-104) after a run of
    sorted, unsorted and duplicated batches (the oracle's FifoRing keeps the
    same per-level counters and is pinned to the reference's rings)."""
    from paper_2112_08541_b200.cachesim import CacheConfig, cold_state, simulate
    from paper_2112_08541_b200.sampler import AccessTrace
    rng = np.random.default_rng(11 + d + cap)
    batches = []
    for i in range(30):
        b = rng.choice(300, size=int(rng.integers(1, 90)), replace=False)
        if i % 3 == 0:
            b = np.sort(b)
        elif i % 3 == 1:
            b = np.concatenate([b, b[: max(1, b.size // 4)]])
        batches.append(b.astype(np.int64))
    cfg = CacheConfig(device_capacity=cap, host_capacity=hcap, num_devices=d, feature_bytes_per_node=16)
    state = cold_state(cfg)
    rep = simulate(AccessTrace(batches=batches), cfg, state=state)
    ref = co.FifoEngine(cap, hcap, d)
    cnt, _ = ref.run(batches)
    assert rep.batch_insertions == cnt[:, 5].tolist() and rep.batch_evictions == cnt[:, 6].tolist()
    for h in range(d):
        lv = state.devices[h]
        assert (lv.insertions, lv.evictions, lv.metadata_updates) == (ref.devices[h].insertions,
                                                                      ref.devices[h].evictions, 0), h
    assert (state.host.insertions, state.host.evictions) == (ref.host.insertions, ref.host.evictions)
