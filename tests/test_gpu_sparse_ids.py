"""GPU parity: sparse / >= 2^31 int64 node IDs.

gnnio's FIFO levels are dicts (cachesim.py:81-107), so its `simulate`
(cachesim.py:275-363) takes any int64 node ID. The B200 path runs such traces
on dense ranks from the open-addressing hash dedup (`bgl_hash_unique`, the
north_star's hash table), with each rank's shard = ID % d
(`bgl_cache_set_home_map`) and resident ranks renamed when the key set grows
(`bgl_cache_remap`). Checked against `tests/golden/sparse.npz` (produced by
gnnio itself, tests/golden/make_golden.py `make_sparse`) and np.unique."""

import numpy as np
import pytest
import torch

from packing import get

from oracle import cache_oracle as co

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
        yield (ci, int(d), int(cap), int(hcap), bd, batches[sl], codes[sl], cnt[sl], dsl[sl], dtl[sl], hsl[sl],
               htl[sl])
        b0 += nb


def _hash_unique(keys: np.ndarray, key_bits: int = 0):
    from paper_2112_08541_b200 import _lib
    lib = _lib.load()
    n = keys.size
    k = torch.from_numpy(keys.astype(np.int64)).cuda()
    ws = torch.empty(int(lib.bgl_hash_unique_workspace(n)), dtype=torch.uint8, device="cuda")
    uniq = torch.full((max(n, 1),), -7, dtype=torch.int64, device="cuda")
    cnt = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    rank = torch.full((max(n, 1),), -1, dtype=torch.int32, device="cuda")
    _lib.check(lib.bgl_hash_unique(k.data_ptr() if n else None, n, key_bits, ws.data_ptr(), uniq.data_ptr(),
                                   cnt.data_ptr(), rank.data_ptr(), _lib.stream_ptr()))
    U = int(cnt.item())
    return uniq[:U].cpu().numpy(), rank[:n].cpu().numpy()


@pytest.mark.parametrize("n,hi,bits", [(0, 1, 0), (1, 10, 0), (1000, 2**62, 62), (50_000, 2**63 - 1, 0),
                                       (200_000, 1000, 10), (1_000_003, 2**40, 40), (300_000, 2**31 + 7, 32)])
def test_hash_unique_matches_np_unique(n, hi, bits):
    rng = np.random.default_rng(n + 3)
    keys = rng.integers(0, hi, size=n, dtype=np.int64)
    if n > 10:
        keys[: n // 10] = keys[n // 10: 2 * (n // 10)]          # duplicates
    u, r = _hash_unique(keys, bits)
    eu, er = np.unique(keys, return_inverse=True)
    assert np.array_equal(u, eu)
    assert np.array_equal(r, er.ravel())


def test_hash_unique_all_equal_and_max_key():
    keys = np.full(70_000, 2**63 - 1, dtype=np.int64)
    keys[::7] = 0
    u, r = _hash_unique(keys)
    assert u.tolist() == [0, 2**63 - 1]
    assert np.array_equal(r, (keys != 0).astype(np.int32))


def test_sparse_whole_trace_matches_reference(golden):
    from paper_2112_08541_b200 import cachesim as cs
    from paper_2112_08541_b200.sampler import AccessTrace
    npz = golden("sparse")
    for ci, d, cap, hcap, bd, batches, codes, cnt, *_ in _cases(npz):
        cfg = cs.CacheConfig(device_capacity=cap, host_capacity=hcap, num_devices=d)
        rep = cs.simulate(AccessTrace(batches=batches), cfg, batch_devices=bd, record_outcomes=True)
        got = [sum(rep.batch_own_hits), sum(rep.batch_peer_hits), sum(rep.batch_host_hits), sum(rep.batch_misses),
               sum(rep.batch_insertions), sum(rep.batch_evictions)]
        assert got == npz["whole"][ci].tolist(), ci
        # whole-trace codes = the batch-at-a-time reference codes (same state sequence)
        assert rep.outcomes == [["DPHM"[c] for c in cd] for cd in codes], ci


def test_sparse_state_every_batch_matches_reference(golden):
    """Batch-at-a-time with a persistent state: every call grows the key set,
    so resident ranks are renamed each time; rings (as IDs), tails, codes and
    counters after every batch equal gnnio's."""
    from paper_2112_08541_b200 import cachesim as cs
    from paper_2112_08541_b200.sampler import AccessTrace
    npz = golden("sparse")
    for ci, d, cap, hcap, bd, batches, codes, cnt, dsl, dtl, hsl, htl in _cases(npz):
        cfg = cs.CacheConfig(device_capacity=cap, host_capacity=hcap, num_devices=d)
        state = cs.cold_state(cfg)
        for i, b in enumerate(batches):
            rep = cs.simulate(AccessTrace(batches=[b]), cfg, batch_devices=[bd[i] if bd else i % d], state=state,
                              record_outcomes=True)
            row = [rep.batch_queries[0], rep.batch_own_hits[0], rep.batch_peer_hits[0], rep.batch_host_hits[0],
                   rep.batch_misses[0], rep.batch_insertions[0], rep.batch_evictions[0],
                   rep.batch_metadata_updates[0]]
            assert row == cnt[i].tolist(), (ci, i)
            assert rep.outcomes[0] == ["DPHM"[c] for c in codes[i]], (ci, i)
            ds, dt, hs, ht = state.engine.export()
            assert np.array_equal(ds.ravel(), dsl[i]), (ci, i)
            assert dt.tolist() == dtl[i].tolist(), (ci, i)
            assert np.array_equal(hs, hsl[i]), (ci, i)
            assert ht == int(htl[i][0]), (ci, i)


def test_dense_state_then_sparse_trace():
    """A state built on dense IDs keeps working when a later trace brings IDs
    >= 2^31 (the dense ranks become keys 0..n-1 of the sparse map)."""
    from paper_2112_08541_b200 import cachesim as cs
    from paper_2112_08541_b200.sampler import AccessTrace
    rng = np.random.default_rng(11)
    dense = [np.unique(rng.integers(0, 500, size=80)) for _ in range(6)]
    sparse = [np.unique(np.concatenate([rng.integers(0, 500, size=40),
                                        rng.integers(2**33, 2**33 + 300, size=40)])) for _ in range(6)]
    for d, cap, hcap in ((1, 60, 0), (3, 25, 16), (4, 10, 64)):
        cfg = cs.CacheConfig(device_capacity=cap, host_capacity=hcap, num_devices=d)
        state = cs.cold_state(cfg)
        oracle = co.FifoEngine(cap, hcap, d)
        for part in (dense, sparse, dense):
            rep = cs.simulate(AccessTrace(batches=part), cfg, state=state, record_outcomes=True)
            c, cd = oracle.run(part, [i % d for i in range(len(part))])
            assert np.array_equal(np.array([rep.batch_queries, rep.batch_own_hits, rep.batch_peer_hits,
                                            rep.batch_host_hits, rep.batch_misses, rep.batch_insertions,
                                            rep.batch_evictions]).T, c)
            assert rep.outcomes == [["DPHM"[x] for x in y] for y in cd]
            ds, _, hs, _ = state.engine.export()
            assert np.array_equal(ds.ravel(), np.concatenate([r.slots for r in oracle.devices]))
            assert np.array_equal(hs, oracle.host.slots)
