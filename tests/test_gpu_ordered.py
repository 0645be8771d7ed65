"""GPU parity: gnnio's LRU and LFU levels (cachesim.py:110-175) through the
drop-in `simulate` (cachesim.py:275-363), bit-exact.

`tests/golden/ordered.npz` was produced by gnnio itself
(tests/golden/make_golden.py `make_ordered`): 48 cases (sorted / unsorted /
duplicated batches, d in {1, 2, 3, 4, 8}, device capacities 0-39, host
levels 0 / 1 / 8 / 30, routed batches), replayed batch by batch on a
persistent state -- counters incl. metadata updates, per-node codes, and
every level after every batch (LRU: `entries` order; LFU: `freq`, `tick_of`,
`tick`) -- plus the desk-scale sampler trace at d = 1, 2, 4. The device runs
the closed forms of `oracle/cache_oracle.py` OrderedLevel
(`bgl_cache_update_ordered`, csrc/ordered.cu)."""

import numpy as np
import pytest

from packing import get

from oracle import cache_oracle as co

pytestmark = pytest.mark.gpu


def _cases(npz):
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
        yield (ci, ("lru", "lfu")[pol], int(d), int(cap), int(hcap), bd, batches[b0:b0 + nb], codes[b0:b0 + nb],
               cnt[b0:b0 + nb], logs[l0:l0 + nl], freqs[l0:l0 + nl], ticks[l0:l0 + nl], lticks[l0:l0 + nl])
        b0 += nb
        l0 += nl


def _row(rep, i=0):
    return [rep.batch_queries[i], rep.batch_own_hits[i], rep.batch_peer_hits[i], rep.batch_host_hits[i],
            rep.batch_misses[i], rep.batch_insertions[i], rep.batch_evictions[i], rep.batch_metadata_updates[i]]


def test_lru_lfu_every_batch_matches_reference(golden):
    from paper_2112_08541_b200 import cachesim as cs
    from paper_2112_08541_b200.sampler import AccessTrace
    npz = golden("ordered")
    for ci, policy, d, cap, hcap, bd, batches, codes, cnt, logs, freqs, ticks, lticks in _cases(npz):
        cfg = cs.CacheConfig(device_capacity=cap, host_capacity=hcap, num_devices=d, policy=policy)
        state = cs.cold_state(cfg)
        for i, b in enumerate(batches):
            rep = cs.simulate(AccessTrace(batches=[b]), cfg, batch_devices=[bd[i] if bd else i % d], state=state,
                              record_outcomes=True)
            assert _row(rep) == cnt[i].tolist(), (ci, policy, i)
            assert rep.outcomes[0] == ["DPHM"[c] for c in codes[i]], (ci, i)
            if ci % 4 and i != len(batches) - 1:
                continue                     # levels read back on a quarter of the cases + every last batch
            for y in range(d + 1):
                lst, fq, tk, lt, _ = state.engine.ordered_level(y)
                k = i * (d + 1) + y
                assert lst.tolist() == logs[k].tolist(), (ci, policy, i, y)
                if policy == "lfu":
                    assert fq.tolist() == freqs[k].tolist(), (ci, i, y)
                    assert tk.tolist() == ticks[k].tolist(), (ci, i, y)
                    assert lt == lticks[k], (ci, i, y)


def test_lru_lfu_whole_trace_and_views(golden):
    """The whole-trace call (one simulate over every batch) gives the same
    counters; the level views mirror the reference attributes."""
    from paper_2112_08541_b200 import cachesim as cs
    from paper_2112_08541_b200.sampler import AccessTrace
    npz = golden("ordered")
    for ci, policy, d, cap, hcap, bd, batches, codes, cnt, logs, freqs, ticks, lticks in _cases(npz):
        if ci % 3:
            continue
        cfg = cs.CacheConfig(device_capacity=cap, host_capacity=hcap, num_devices=d, policy=policy)
        state = cs.cold_state(cfg)
        rep = cs.simulate(AccessTrace(batches=batches), cfg, batch_devices=bd, state=state, record_outcomes=True)
        got = np.array([_row(rep, i) for i in range(len(batches))])
        assert np.array_equal(got, cnt), (ci, policy)
        last = (len(batches) - 1) * (d + 1)
        for y, lv in enumerate(list(state.devices) + [state.host]):
            assert len(lv) == logs[last + y].size
            if policy == "lru":
                assert list(lv.entries.keys()) == logs[last + y].tolist()
            else:
                assert lv.freq == dict(zip(logs[last + y].tolist(), freqs[last + y].tolist()))
                assert lv.tick == lticks[last + y]
        assert sum(lv.insertions for lv in list(state.devices) + [state.host]) == int(cnt[:, 5].sum())
        assert sum(lv.evictions for lv in list(state.devices) + [state.host]) == int(cnt[:, 6].sum())
        assert sum(lv.metadata_updates for lv in list(state.devices) + [state.host]) == int(cnt[:, 7].sum())


def test_lru_lfu_real_trace(golden):
    from paper_2112_08541_b200 import cachesim as cs
    from paper_2112_08541_b200.sampler import AccessTrace
    npz = golden("ordered")
    trace = AccessTrace(batches=get(npz, "real_trace"))
    for j, (policy, d) in enumerate([(p, d) for p in ("lru", "lfu") for d in (1, 2, 4)]):
        rep = cs.simulate(trace, cs.CacheConfig(device_capacity=500 // d, host_capacity=250, num_devices=d,
                                                policy=policy))
        got = np.array([rep.batch_queries, rep.batch_own_hits, rep.batch_peer_hits, rep.batch_host_hits,
                        rep.batch_misses, rep.batch_insertions, rep.batch_evictions, rep.batch_metadata_updates])
        assert np.array_equal(got, npz["real_counters"][j]), (policy, d)


@pytest.mark.parametrize("policy", ["lru", "lfu"])
def test_lru_lfu_large_vs_oracle(policy):
    """Levels of 20K-60K residents (several CTA chunks per level) and 8 shards
    + a host level, against the batch-parallel oracle."""
    from paper_2112_08541_b200 import cachesim as cs
    from paper_2112_08541_b200.sampler import AccessTrace
    rng = np.random.default_rng(3)
    batches = [np.unique(rng.integers(0, 400_000, size=60_000) ** 1 // (1 + (k % 3))) for k in range(6)]
    batches += [rng.integers(0, 150_000, size=40_000) for _ in range(3)]          # unsorted with duplicates
    for d, cap, hcap in ((1, 60_000, 0), (8, 2_500, 20_000)):
        cfg = cs.CacheConfig(device_capacity=cap, host_capacity=hcap, num_devices=d, policy=policy)
        rep = cs.simulate(AccessTrace(batches=batches), cfg, record_outcomes=True)
        c, cd, _ = co.simulate_ordered(policy, batches, cap, hcap, d)
        got = np.array([_row(rep, i) for i in range(len(batches))])
        assert np.array_equal(got, c), (policy, d)
        assert rep.outcomes == [["DPHM"[x] for x in y] for y in cd]


@pytest.mark.parametrize("policy", ["lru", "lfu"])
def test_lru_lfu_sparse_ids(policy):
    """Sparse int64 IDs (>= 2^31) on LRU / LFU: the per-node state follows its
    residents when the key set grows between calls."""
    from paper_2112_08541_b200 import cachesim as cs
    from paper_2112_08541_b200.sampler import AccessTrace
    rng = np.random.default_rng(9)
    universe = np.unique(rng.integers(2**33, 2**40, size=400))
    parts = [[rng.choice(universe[: 100 * (k + 1)], size=60) for _ in range(4)] for k in range(4)]
    for d, cap, hcap in ((1, 40, 0), (3, 12, 20)):
        cfg = cs.CacheConfig(device_capacity=cap, host_capacity=hcap, num_devices=d, policy=policy)
        state = cs.cold_state(cfg)
        ost = None
        for part in parts:
            rep = cs.simulate(AccessTrace(batches=part), cfg, state=state, record_outcomes=True)
            c, cd, ost = co.simulate_ordered(policy, part, cap, hcap, d, state=ost)
            got = np.array([_row(rep, i) for i in range(len(part))])
            assert np.array_equal(got, c)
            assert rep.outcomes == [["DPHM"[x] for x in y] for y in cd]
            for y, lv in enumerate(list(ost[0]) + [ost[1]]):
                assert state.engine.ordered_level(y)[0].tolist() == lv.log
