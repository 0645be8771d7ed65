"""GPU parity: sampler + dedup/relabel vs the reference's golden vectors and
the CPU oracle (bit-exact)."""

import numpy as np
import pytest
import torch

from conftest import golden_graph
from packing import get

from oracle import pcg64
from oracle import sampler_oracle as so

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bgl():
    import paper_2112_08541_b200 as p
    return p


class G:
    """Minimal graph object (duck-typed like gnnio.graph.Graph)."""

    def __init__(self, off, col, train=None):
        self.row_offsets = off
        self.col_indices = col
        self.num_nodes = len(off) - 1
        self.train_mask = train if train is not None else np.zeros(self.num_nodes, bool)


def test_pcg64_draws_bit_exact(bgl):
    from paper_2112_08541_b200 import _lib
    from paper_2112_08541_b200.sampler import pcg_states, pcg_tables
    tables = pcg_tables(pcg_states(7, [3, 4]))
    ref = np.random.default_rng((7, 3)).random(5000)
    out = torch.empty(300, dtype=torch.int64, device="cuda")
    for first in (0, 1, 4700):
        _lib.call("bgl_pcg64_draws", tables[0].data_ptr(), first, 300, out.data_ptr(), _lib.stream_ptr())
        m = out.cpu().numpy().view(np.uint64)
        assert np.array_equal(m.astype(np.float64) * 2.0 ** -53, ref[first:first + 300])
    st, inc = pcg64.stream_state((7, 4))
    assert np.array_equal(tables[1].cpu().numpy().view(np.uint64), pcg64.jump_table(st, inc))


def test_sample_batch_matches_reference_golden(golden, bgl):
    npz = golden("sampler")
    meta = npz["case_meta"]
    seeds = get(npz, "case_seeds")
    fans = get(npz, "case_fanouts")
    ids = get(npz, "hop_ids")
    dist = get(npz, "distinct")
    names = list(npz["graph_names"])
    h = 0
    for c in range(len(meta)):
        gi, seed, bseed = (int(x) for x in meta[c])
        off, col, train = golden_graph(npz, names[gi])
        g = G(off, col, train)
        fan = tuple(int(f) for f in fans[c])
        cfg = bgl.SamplingConfig(fanouts=fan, seed=seed)
        fr, distinct = bgl.sample_batch(g, seeds[c], cfg, batch_seed=bseed)
        for k in range(len(fan)):
            assert np.array_equal(fr[k], ids[h + k]), (c, k)
        assert np.array_equal(distinct, dist[c])
        h += len(fan)


def test_relabelled_subgraph_matches_unique_inverse(golden, bgl):
    from paper_2112_08541_b200.sampler import sample_batch_relabelled
    npz = golden("sampler")
    off, col, train = golden_graph(npz, "dense")
    g = G(off, col, train)
    seeds = np.flatnonzero(train)[:50]
    cfg = bgl.SamplingConfig(fanouts=(15, 10, 5), seed=3)
    distinct, edges, _ = sample_batch_relabelled(g, seeds, cfg, batch_seed=9)
    fr, pidx, d_ref, inv = so.sample_batch(off, col, seeds, cfg.fanouts, 3, 9)
    assert np.array_equal(distinct.cpu().numpy(), d_ref)
    lens = [len(seeds)] + [len(f) for f in fr]
    starts = np.concatenate([[0], np.cumsum(lens)])
    for h, (src, dst) in enumerate(edges):
        par_local = inv[starts[h]:starts[h + 1]][pidx[h]]
        child_local = inv[starts[h + 1]:starts[h + 2]]
        assert np.array_equal(src.cpu().numpy(), par_local)
        assert np.array_equal(dst.cpu().numpy(), child_local)


def test_simulate_epoch_matches_reference_golden(golden, bgl):
    npz = golden("sampler")
    off, col, train = golden_graph(npz, "planted")
    g = G(off, col, train)

    class P:
        pass

    for e, (k, seed, nb) in enumerate(npz["epoch_meta"]):
        p = P()
        p.part_of = npz[f"epoch{e}_part_of"]
        p.k = int(k)
        sched = bgl.BatchSchedule(batches=get(npz, f"epoch{e}_batches"), batch_size=0, policy="x")
        fans = tuple(int(x) for x in npz[f"epoch{e}_fanouts"])
        trace, rep = bgl.simulate_epoch(g, p, sched, bgl.SamplingConfig(fanouts=fans, seed=int(seed)))
        ref = get(npz, f"epoch{e}_trace")
        assert len(trace.batches) == nb
        assert all(np.array_equal(a, b) for a, b in zip(trace.batches, ref))
        assert [rep.local_accesses, rep.remote_accesses] == npz[f"epoch{e}_local_remote"].tolist()
        assert np.array_equal(rep.seed_load, npz[f"epoch{e}_seed_load"])
        assert np.array_equal(rep.request_load, npz[f"epoch{e}_request_load"])


def test_edge_cases(bgl):
    # star: hop 2 from the three sampled leaves is the centre three times
    off = np.array([0, 5, 6, 7, 8, 9, 10])
    col = np.array([1, 2, 3, 4, 5, 0, 0, 0, 0, 0])
    g = G(off, col)
    fr, d = bgl.sample_batch(g, np.array([0]), bgl.SamplingConfig(fanouts=(3, 3), seed=7))
    assert fr[1].tolist() == [0, 0, 0]
    with pytest.raises(ValueError):
        bgl.sample_batch(g, np.empty(0, np.int64), bgl.SamplingConfig())
    # isolated seed contributes nothing
    off2 = np.array([0, 1, 2, 2])
    col2 = np.array([1, 0])
    fr, d = bgl.sample_batch(G(off2, col2), np.array([2]), bgl.SamplingConfig(fanouts=(4, 4)))
    assert len(fr[0]) == 0 and len(fr[1]) == 0 and d.tolist() == [2]


@pytest.mark.parametrize("fanouts", [(15, 10, 5), (25, 10), (40,), (3, 3, 3, 3), (32, 2), (1, 1, 1)])
def test_random_power_law_matches_oracle(bgl, fanouts):
    from paper_2112_08541_b200.graph import generate_power_law_device
    dg = generate_power_law_device(30000, 24, seed=5, train_fraction=0.1, num_labels=8)
    hg = dg.to_host()
    rng = np.random.default_rng(1)
    train = hg.train_nodes()
    for bseed in (0, 17):
        seeds = train[rng.integers(len(train), size=256)]
        cfg = bgl.SamplingConfig(fanouts=fanouts, seed=11)
        fr, d = bgl.sample_batch(dg, seeds, cfg, batch_seed=bseed)
        fr_o, _, d_o, _ = so.sample_batch(hg.row_offsets, hg.col_indices, seeds, fanouts, 11, bseed)
        for a, b in zip(fr, fr_o):
            assert np.array_equal(a, b)
        assert np.array_equal(d, d_o)


@pytest.mark.parametrize("fanouts", [(5, 5), (32,), (12, 3)])
def test_hubs_zero_degree_and_duplicates_match_oracle(bgl, fanouts):
    """Parents the flat-stream kernel must route elsewhere or skip: hubs with
    deg > 2048 (CTA kernel) sitting between light parents of the same run,
    isolated (deg 0) parents, parents repeated in a hop, deg == fanout."""
    rng = np.random.default_rng(3)
    n = 12000
    adj = [set() for _ in range(n)]
    for h in (5, 6, 900):                       # three hubs, two adjacent IDs
        for v in rng.choice(n, size=3000 + h, replace=False):
            if v != h:
                adj[h].add(int(v)); adj[int(v)].add(h)
    for v in range(20, n - 1):                  # chain + random extra edges; 0..19 isolated
        if v % 7:
            adj[v].add(v + 1); adj[v + 1].add(v)
        u = int(rng.integers(20, n))
        if u != v:
            adj[v].add(u); adj[u].add(v)
    for v in range(20):
        for u in list(adj[v]):
            adj[u].discard(v)
        adj[v] = set()
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum([len(a) for a in adj])
    col = np.concatenate([np.array(sorted(a), np.int64) for a in adj])
    g = G(off, col)
    seeds = np.concatenate([np.array([5, 6, 900, 0, 3, 5, 5, 6]), rng.integers(0, n, 500)])
    for bseed in (1, 2):
        cfg = bgl.SamplingConfig(fanouts=fanouts, seed=4)
        fr, d = bgl.sample_batch(g, seeds, cfg, batch_seed=bseed)
        fr_o, _, d_o, _ = so.sample_batch(off, col, seeds, fanouts, 4, bseed)
        for a, b in zip(fr, fr_o):
            assert np.array_equal(a, b)
        assert np.array_equal(d, d_o)


def test_exact_generator_device_csr_matches_reference(golden, bgl):
    """generate_power_law (native edges + device CSR) == gnnio's graphs."""
    npz = golden("graphgen")
    for i, ((n, d, seed, nl), (tf, cf)) in enumerate(zip(npz["specs"], npz["fracs"])):
        g = bgl.generate_power_law(int(n), int(d), int(seed), float(tf), int(nl), float(cf))
        assert np.array_equal(g.row_offsets, npz[f"off_{i}"]) and np.array_equal(g.col_indices, npz[f"col_{i}"])
        assert np.array_equal(g.train_mask, np.unpackbits(npz[f"train_{i}"])[:int(n)].astype(bool))
        assert np.array_equal(g.labels, npz[f"labels_{i}"].astype(np.int64))


def test_device_csr_chunked_by_source_range():
    """csr_from_edges_device with tiny passes (the papers100M path: CUB sorts
    < 2^31 keys) equals the single-pass CSR and numpy's csr_from_edges."""
    from oracle import graph_oracle as go
    from paper_2112_08541_b200.graph import csr_from_edges_device, power_law_edges
    edges, _, _ = power_law_edges(5000, 12, 4, 0.1, 3)
    off, col = go.csr_from_edges(edges.astype(np.int64), 5000)
    for mk in (1 << 29, 4096, 1000):
        ip, ix = csr_from_edges_device(edges, 5000, max_keys=mk)
        assert np.array_equal(ip.cpu().numpy(), off) and np.array_equal(ix.cpu().numpy(), col), mk
