"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py). CPU only."""

import numpy as np
import pytest

from conftest import golden_graph
from packing import get

from oracle import cache_oracle as co
from oracle import features_oracle as fo
from oracle import ordering_oracle as oo
from oracle import pcg64
from oracle import sampler_oracle as so


def _cases(npz):
    meta = npz["case_meta"]
    seeds = get(npz, "case_seeds")
    fans = get(npz, "case_fanouts")
    ids = get(npz, "hop_ids")
    pidx = get(npz, "hop_pidx")
    dist = get(npz, "distinct")
    names = list(npz["graph_names"])
    h = 0
    for c in range(len(meta)):
        gi, seed, bseed = (int(x) for x in meta[c])
        nh = len(fans[c])
        yield names[gi], seeds[c], tuple(int(f) for f in fans[c]), seed, bseed, ids[h:h + nh], pidx[h:h + nh], dist[c]
        h += nh


@pytest.mark.parametrize("hop", [so.sample_hop, so.sample_hop_topk], ids=["segsort", "topk"])
def test_sampler_matches_reference(golden, hop):
    npz = golden("sampler")
    n = 0
    for gname, seeds, fans, seed, bseed, ids, pidx, dist in _cases(npz):
        off, col, _ = golden_graph(npz, gname)
        fr, pi, distinct, inverse = so.sample_batch(off, col, seeds, fans, seed, bseed, hop=hop)
        for a, b in zip(fr, ids):
            assert np.array_equal(a, b)
        for a, b in zip(pi, pidx):
            assert np.array_equal(a, b)
        assert np.array_equal(distinct, dist)
        allk = np.concatenate([seeds] + fr)
        assert np.array_equal(distinct[inverse], allk)
        n += 1
    assert n >= 14


def test_epochs_match_reference(golden):
    npz = golden("sampler")
    off, col, _ = golden_graph(npz, "planted")
    for e, (k, seed, nb) in enumerate(npz["epoch_meta"]):
        batches = get(npz, f"epoch{e}_batches")
        fans = tuple(int(x) for x in npz[f"epoch{e}_fanouts"])
        trace, local, remote, sl, rl = so.simulate_epoch(off, col, npz[f"epoch{e}_part_of"], int(k), batches, fans, int(seed))
        ref = get(npz, f"epoch{e}_trace")
        assert len(trace) == nb == len(ref)
        assert all(np.array_equal(a, b) for a, b in zip(trace, ref))
        assert [local, remote] == npz[f"epoch{e}_local_remote"].tolist()
        assert np.array_equal(sl, npz[f"epoch{e}_seed_load"])
        assert np.array_equal(rl, npz[f"epoch{e}_request_load"])


def test_pcg64_restatement_matches_numpy():
    st, inc = pcg64.stream_state((7, 3))
    ref = np.random.default_rng((7, 3)).random(2000)
    for i in (0, 1, 2, 5, 999, 1999):
        assert pcg64.draw_u53(st, inc, i) * 2.0 ** -53 == ref[i]
    table = pcg64.jump_table(st, inc)
    assert table.shape == (pcg64.TABLE_ROWS, 4)
    # composing one map per nonzero hex digit equals advance()
    delta = 0x3B0A07
    s = st
    for i in range(6):
        j = (delta >> (4 * i)) & 15
        if j:
            r = 1 + 15 * i + (j - 1)
            a = (int(table[r, 0]) << 64) | int(table[r, 1])
            c = (int(table[r, 2]) << 64) | int(table[r, 3])
            s = (a * s + c) & pcg64.MASK128
    assert s == pcg64.advance(st, inc, delta)


def _cache_cases(npz):
    specs = npz["specs"]
    batches = get(npz, "batches")
    codes = get(npz, "codes")
    dslots = get(npz, "dev_slots")
    dtails = get(npz, "dev_tails")
    hslots = get(npz, "host_slots")
    htails = get(npz, "host_tails")
    cnt = npz["counters"]
    b0 = 0
    for ci, (d, cap, hcap, nb, use_bd, kind) in enumerate(specs):
        bd = npz[f"bd_{ci}"].tolist() if use_bd else None
        sl = slice(b0, b0 + nb)
        yield (int(d), int(cap), int(hcap), bd, batches[sl], codes[sl], cnt[sl], dslots[sl], dtails[sl],
               hslots[sl], htails[ci], int(kind))
        b0 += nb


def test_fifo_sequential_oracle_matches_reference(golden):
    npz = golden("cache")
    for d, cap, hcap, bd, batches, codes, cnt, dsl, dtl, hsl, htl, _ in _cache_cases(npz):
        eng = co.FifoEngine(cap, hcap, d)
        for i, b in enumerate(batches):
            c, cd = eng.run([b], [bd[i] if bd else i % d])
            assert np.array_equal(cd[0], codes[i])
            assert np.array_equal(c[0], cnt[i][:7])
            assert cnt[i][7] == 0   # FIFO never updates metadata (cachesim.py:49, 94-104)
            assert np.array_equal(np.concatenate([r.slots for r in eng.devices]) if cap else np.empty(0), dsl[i])
            assert [r.tail for r in eng.devices] == dtl[i].tolist()
            assert np.array_equal(eng.host.slots, hsl[i])
            assert eng.host.tail == htl[i]


def test_fifo_batched_oracle_matches_reference(golden):
    npz = golden("cache")
    for d, cap, hcap, bd, batches, codes, cnt, dsl, dtl, hsl, htl, _ in _cache_cases(npz):
        state = None
        for i, b in enumerate(batches):
            kw = {} if state is None else dict(dev_slots=state[0], dev_tails=state[1], host_slots=state[2], host_tail=state[3])
            c, cd, state = co.simulate_batched([b], cap, hcap, d, [bd[i] if bd else i % d], **kw)
            assert np.array_equal(cd[0], codes[i])
            assert np.array_equal(c[0], cnt[i][:7])
            assert np.array_equal(state[0].ravel(), dsl[i])
            assert state[1].tolist() == dtl[i].tolist()
            assert np.array_equal(state[2], hsl[i])
            assert state[3] == htl[i]


def test_fifo_sparse_ids_oracle_matches_reference(golden):
    """Sparse / >= 2^31 int64 IDs (tests/golden/sparse.npz, gnnio's dict FIFO):
    the sequential oracle restates them exactly, so the GPU tests can use it."""
    npz = golden("sparse")
    for d, cap, hcap, bd, batches, codes, cnt, dsl, dtl, hsl, htl, _ in _cache_cases(npz):
        eng = co.FifoEngine(cap, hcap, d)
        for i, b in enumerate(batches):
            c, cd = eng.run([b], [bd[i] if bd else i % d])
            assert np.array_equal(cd[0], codes[i])
            assert np.array_equal(c[0], cnt[i][:7])
            assert np.array_equal(np.concatenate([r.slots for r in eng.devices]) if cap else np.empty(0), dsl[i])
            assert np.array_equal(eng.host.slots, hsl[i])
    assert npz["batches__data"].max() >= 2**40 and npz["batches__data"].min() >= 0


def _ordered_cases(npz):
    specs = npz["specs"]
    batches = get(npz, "batches")
    codes = get(npz, "codes")
    logs, freqs, ticks = get(npz, "logs"), get(npz, "freqs"), get(npz, "ticks")
    lticks = npz["level_ticks"]
    cnt = npz["counters"]
    b0 = l0 = 0
    for ci, (d, cap, hcap, nb, use_bd, kind, pol) in enumerate(specs):
        bd = npz[f"bd_{ci}"].tolist() if use_bd else None
        nl = nb * (d + 1)
        yield (("lru", "lfu")[pol], int(d), int(cap), int(hcap), bd, batches[b0:b0 + nb], codes[b0:b0 + nb],
               cnt[b0:b0 + nb], logs[l0:l0 + nl], freqs[l0:l0 + nl], ticks[l0:l0 + nl], lticks[l0:l0 + nl])
        b0 += nb
        l0 += nl


def test_lru_lfu_batched_oracle_matches_reference(golden):
    """The batch-parallel LRU / LFU closed forms (oracle/cache_oracle.py
    OrderedLevel, what the CUDA update implements) against gnnio's
    sequential levels (tests/golden/ordered.npz): counters incl. metadata
    updates, codes, and every level's order / freq / ticks after every batch."""
    npz = golden("ordered")
    for policy, d, cap, hcap, bd, batches, codes, cnt, logs, freqs, ticks, lticks in _ordered_cases(npz):
        state = None
        for i, b in enumerate(batches):
            c, cd, state = co.simulate_ordered(policy, [b], cap, hcap, d, [bd[i] if bd else i % d], state=state)
            assert np.array_equal(cd[0], codes[i])
            assert np.array_equal(c[0], cnt[i])
            for y, lv in enumerate(list(state[0]) + [state[1]]):
                k = i * (d + 1) + y
                assert lv.log == logs[k].tolist(), (policy, i, y)
                if policy == "lfu":
                    assert [lv.freq[v] for v in lv.log] == freqs[k].tolist()
                    assert [lv.tick_of[v] for v in lv.log] == ticks[k].tolist()
                    assert lv.tick == lticks[k]
    real = get(npz, "real_trace")
    for j, (policy, d) in enumerate([(p, d) for p in ("lru", "lfu") for d in (1, 2, 4)]):
        c, _, _ = co.simulate_ordered(policy, real, 500 // d, 250, d)
        assert np.array_equal(c.T, npz["real_counters"][j])


def test_fifo_real_trace(golden):
    npz = golden("cache")
    trace = get(npz, "real_trace")
    for j, d in enumerate((1, 2, 4, 8)):
        c, _, _ = co.simulate_batched(trace, 500 // d, 250, d)
        assert np.array_equal(c.T, npz["real_counters"][j])


def test_ordering_matches_reference(golden):
    npz = golden("ordering")
    names = list(npz["graph_names"])
    seqs = get(npz, "seqs")
    s0 = 0
    for gi, S, seed in npz["seq_meta"]:
        gname = names[gi] if gi < 100 else f"rnd{gi - 100}"
        off, col, train = golden_graph(npz, gname)
        res = oo.bfs_sequences(off, col, train, int(S), int(seed))
        assert len(res) == S
        for a, b in zip(res, seqs[s0:s0 + S]):
            assert np.array_equal(a, b)
        s0 += S
    batches = get(npz, "sched_batches")
    b0 = 0
    for gi, S, b, seed, nb, kind in npz["sched_meta"]:
        gname = names[gi] if gi < 100 else f"rnd{gi - 100}"
        off, col, train = golden_graph(npz, gname)
        if kind == 0:
            got = oo.proximity_schedule(off, col, train, int(S), int(b), int(seed))
        else:
            got = oo.random_schedule(train, int(b), int(seed))
        assert len(got) == nb
        for x, y in zip(got, batches[b0:b0 + nb]):
            assert np.array_equal(x, y)
        b0 += nb


def test_interleave_hand_cases():
    # ordering tests test_form_batches_* (test_ordering.py:113-128 of the reference)
    assert [b.tolist() for b in oo.interleave([np.arange(7)], 3)[1]] == [[0, 1, 2], [3, 4, 5], [6]]
    assert [b.tolist() for b in oo.interleave([np.array([1, 2]), np.array([3, 4])], 2)[1]] == [[1, 3], [2, 4]]
    assert oo.interleave([np.array([1, 2, 5]), np.array([3])], 2)[1][0].tolist() == [1, 3]
    with pytest.raises(ValueError):
        oo.interleave([np.array([1])], 0)


def test_feature_hash_properties():
    a = fo.synthetic_features(np.array([0, 1, 123456789]), 100, seed=3)
    assert a.dtype == np.float32 and a.shape == (3, 100)
    assert np.all(a >= -0.5) and np.all(a < 0.5)
    assert np.array_equal(a, fo.synthetic_features(np.array([0, 1, 123456789]), 100, seed=3))
    assert not np.array_equal(a, fo.synthetic_features(np.array([0, 1, 123456789]), 100, seed=4))


def _static_cases(npz):
    names = list(npz["graph_names"])
    dev_sets = get(npz, "dev_sets")
    host_sets = get(npz, "host_sets")
    batches = get(npz, "batches")
    codes = get(npz, "codes")
    cnt = npz["counters"]
    di = b0 = 0
    for ci, (gi, d, cap, hcap, nb) in enumerate(npz["meta"]):
        yield (names[gi], int(d), int(cap), int(hcap), dev_sets[di:di + d], host_sets[ci], batches[b0:b0 + nb],
               codes[b0:b0 + nb], cnt[b0:b0 + nb])
        di += d
        b0 += nb


def test_static_oracle_matches_reference(golden):
    npz = golden("static")
    for gname, d, cap, hcap, dsets, hset, batches, codes, cnt in _static_cases(npz):
        off, _, _ = golden_graph(npz, gname)
        dev, host = co.static_warm(off, cap, hcap, d)
        assert [sorted(x.tolist()) for x in dev] == [x.tolist() for x in dsets]
        assert sorted(host.tolist()) == hset.tolist()
        c, cd = co.static_run(batches, dev, host, d)
        assert np.array_equal(c, cnt)
        assert all(np.array_equal(a, b) for a, b in zip(cd, codes))


def _graphgen_cases(npz):
    for i, ((n, d, seed, nl), (tf, cf)) in enumerate(zip(npz["specs"], npz["fracs"])):
        train = np.unpackbits(npz[f"train_{i}"])[:n].astype(bool)
        yield (int(n), int(d), int(seed), float(tf), int(nl), float(cf)), npz[f"off_{i}"], npz[f"col_{i}"], train, \
            npz[f"labels_{i}"].astype(np.int64)


def test_graph_generator_restatement_matches_reference(golden):
    """oracle/graph_oracle.py (numpy PCG64/Lemire/choice + CPython set order)
    reproduces gnnio.graph.generate_power_law exactly (graph.py:218-297)."""
    from oracle import graph_oracle as go
    npz = golden("graphgen")
    for (n, d, seed, tf, nl, cf), off, col, train, labels in _graphgen_cases(npz):
        if n > 5000:
            continue                      # the pure-Python restatement is slow; native covers all cases
        e, lab, tr = go.power_law_edges(n, d, seed, tf, nl, cf)
        o, c = go.csr_from_edges(e, n)
        assert np.array_equal(o, off) and np.array_equal(c, col), (n, d, seed)
        assert np.array_equal(lab, labels)
        assert np.array_equal(tr, np.flatnonzero(train))


def test_oracle_reproduces_reference_c1_epoch(golden):
    """BASELINE.json configs[0] at full size: the reference's own epoch
    (tests/golden/c1.npz: graph, proximity schedule, trace, FIFO outcomes)
    reproduced by the oracle restatement on the native generator's graph."""
    from oracle import cache_oracle as co
    from oracle import graph_oracle as go
    from oracle import ordering_oracle as oo
    from oracle import sampler_oracle as so
    from paper_2112_08541_b200.graph import power_law_edges
    npz = golden("c1")
    n = 100_000
    edges, train, _ = power_law_edges(n, 20, 1, 0.1, 64)
    off, col = go.csr_from_edges(edges.astype(np.int64), n)
    assert len(col) == int(npz["csr_entries"][0])
    sched = oo.proximity_schedule(off, col, train, 4, 1024, 1)
    ref_sched = get(npz, "schedule")
    assert all(np.array_equal(a, b) for a, b in zip(sched, ref_sched))
    trace = [so.sample_batch(off, col, b, (10, 5), 1, i)[2] for i, b in enumerate(sched)]
    ref_trace = get(npz, "trace")
    assert all(np.array_equal(a, b) for a, b in zip(trace, ref_trace))
    cnt, codes = co.FifoEngine(10_000, 0, 1).run(trace)
    assert np.array_equal(cnt, npz["counters"])
    assert all(np.array_equal(a, b) for a, b in zip(codes, get(npz, "codes")))


def test_graph_generator_c_restatement_matches_reference(golden):
    """oracle/powerlaw_ref.c (the C restatement bench.py's reference arm builds
    its graph with) reproduces gnnio.graph.generate_power_law on every golden
    graph, including the ones too large for the pure-Python restatement."""
    from oracle import graph_oracle as go
    npz = golden("graphgen")
    for (n, d, seed, tf, nl, cf), off, col, train, labels in _graphgen_cases(npz):
        o, c, tr, lab = go.generate_power_law_c(n, d, seed, tf, nl, cf)
        assert np.array_equal(o, off) and np.array_equal(c, col), (n, d, seed)
        assert np.array_equal(tr, train), (n, d, seed)
        assert np.array_equal(lab, labels), (n, d, seed)


def test_graph_generator_c_restatement_c2_checksum(golden):
    """BASELINE.json configs[1]: the C restatement's products-shaped graph has
    the CSR size, checksum and offsets tail of the graph gnnio generated
    (tests/golden/c2.npz; ~10 minutes of reference CPU time, seconds here)."""
    from oracle import graph_oracle as go
    npz = golden("c2")
    off, col, train, _ = go.generate_power_law_c(2_400_000, 51, 1, 0.08, 47)
    assert col.size == int(npz["csr_entries"][0])
    assert int((col * (np.arange(col.size) % 1000003 + 1)).sum() % (1 << 61)) == int(npz["csr_checksum"][0])
    assert np.array_equal(off[-1000:], npz["offsets_tail"])
    assert int(train.sum()) == int(0.08 * 2_400_000)
