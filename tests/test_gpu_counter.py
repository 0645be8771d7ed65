"""Counter-RNG sampler mode (SamplingConfig(rng="counter"): Philox4x32-10 +
Floyd's algorithm, csrc/sampler_counter.cu). It is not the reference's numpy
stream, so it is validated the way the north_star asks -- neighbour validity
and fanout distribution -- and bit for bit against its own CPU restatement
(oracle/counter_sampler.py); the cache/gather downstream stays exact for the
trace it produces."""

import numpy as np
import pytest
import torch
from scipy import stats

from oracle import cache_oracle as co
from oracle import counter_sampler as cso
from oracle import features_oracle as fo

pytestmark = pytest.mark.gpu


class G:
    def __init__(self, off, col, train=None):
        self.row_offsets, self.col_indices, self.num_nodes = off, col, len(off) - 1
        self.train_mask = train if train is not None else np.zeros(self.num_nodes, bool)


@pytest.fixture(scope="module")
def graph():
    from paper_2112_08541_b200.graph import generate_power_law_exact_device
    dg = generate_power_law_exact_device(30000, 24, seed=5, train_fraction=0.1, num_labels=8)
    return dg, dg.to_host()


@pytest.mark.parametrize("fanouts", [(15, 10, 5), (25, 10), (32,), (1, 1, 1), (3, 3, 3, 3), (2, 7)])
def test_counter_sampler_matches_its_restatement(graph, fanouts):
    import paper_2112_08541_b200 as bgl
    dg, hg = graph
    rng = np.random.default_rng(2)
    seeds = hg.train_nodes()[rng.integers(hg.num_train(), size=200)]
    for bseed in (0, 9):
        cfg = bgl.SamplingConfig(fanouts=fanouts, seed=11, rng="counter")
        fr, d = bgl.sample_batch(dg, seeds, cfg, batch_seed=bseed)
        fr_o, _, d_o = cso.sample_batch(hg.row_offsets, hg.col_indices, seeds, fanouts, 11, bseed)
        for a, b in zip(fr, fr_o):
            assert np.array_equal(a, b)
        assert np.array_equal(d, d_o)


def test_counter_sampler_neighbour_validity(graph):
    """Every sample is a neighbour of its parent, no parent repeats a neighbour,
    each parent emits min(fanout, deg) samples, parent_idx points back."""
    from paper_2112_08541_b200.sampler import BatchSampler, pcg_states, pcg_tables
    dg, hg = graph
    off, col = hg.row_offsets, hg.col_indices
    s = BatchSampler(dg, (15, 10, 5), 1024, rng="counter")
    seeds = hg.train_nodes()[:1024]
    s.load_seeds(torch.from_numpy(seeds.astype(np.int32)).cuda())
    s.run(pcg_tables(pcg_states(3, [4]))[0])
    counts = s.host_counts()
    parents = seeds.astype(np.int64)
    for h, f in enumerate((15, 10, 5)):
        ids = s.frontier(h, counts).cpu().numpy().astype(np.int64)
        pidx = s.parent_idx(h, counts).cpu().numpy().astype(np.int64)
        deg = off[parents + 1] - off[parents]
        assert len(ids) == int(np.minimum(deg, f).sum())
        assert np.all(np.diff(pidx) >= 0)
        for q in np.unique(pidx):
            mine = ids[pidx == q]
            p = parents[q]
            nb = col[off[p]:off[p + 1]]
            assert len(mine) == min(f, len(nb)) and len(np.unique(mine)) == len(mine)
            assert np.isin(mine, nb).all()
        parents = ids


@pytest.mark.parametrize("hop", [0, 1])
@pytest.mark.parametrize("deg,f", [(20, 5), (9, 6)])
def test_counter_sampler_subsets_are_uniform(deg, f, hop):
    """A hub of degree `deg` sampled with fanout f by 6000 independent parent
    positions: every neighbour appears with probability f/deg and every pair
    with probability C(deg-2, f-2)/C(deg, f) (chi-square, p > 1e-5). hop 0
    runs the sub-warp rejection kernel ((9, 6): the complement branch, 3
    excluded indices drawn), hop 1 the lane-per-parent Floyd kernel (the hub
    reached through a degree-1 node)."""
    import paper_2112_08541_b200 as bgl
    reps = 6000
    # nodes: 0 = hub, 1..deg = its leaves, deg+1 = a node whose only neighbour is the hub
    adj = [list(range(1, deg + 1)) + [deg + 1]] + [[0] for _ in range(deg)] + [[0]]
    if hop == 0:
        adj[0] = list(range(1, deg + 1))
        adj = adj[:deg + 1]
    off = np.concatenate([[0], np.cumsum([len(a) for a in adj])]).astype(np.int64)
    col = np.concatenate([np.array(a, dtype=np.int64) for a in adj])
    g = G(off, col)
    if hop == 0:
        seeds, fans = np.zeros(reps, dtype=np.int64), (f,)
    else:
        seeds, fans = np.full(reps, deg + 1, dtype=np.int64), (1, f)
        deg += 1          # the hub's adjacency also holds the entry node (id deg+1)
    fr, _ = bgl.sample_batch(g, seeds, bgl.SamplingConfig(fanouts=fans, seed=1, rng="counter"))
    picks = fr[hop].reshape(reps, f)
    picks = np.where(picks == deg, 0, picks) if hop else picks - 1   # map neighbour IDs to 0..deg-1
    single = np.bincount(picks.ravel(), minlength=deg)
    assert stats.chisquare(single).pvalue > 1e-5
    pair = np.zeros((deg, deg), dtype=np.int64)
    for row in picks:
        for a in row:
            for b in row:
                if a < b:
                    pair[a, b] += 1
    obs = pair[np.triu_indices(deg, 1)]
    assert stats.chisquare(obs).pvalue > 1e-5


@pytest.mark.parametrize("where", ["host", "hbm"])
def test_counter_pipeline_cache_and_rows_exact(graph, where):
    """Counter-mode pipeline: the trace equals the restatement's, and codes,
    counters and rows equal the FIFO oracle + F[ids] on that trace."""
    from paper_2112_08541_b200.cachesim import CacheConfig
    from paper_2112_08541_b200.features import synthetic_features
    from paper_2112_08541_b200.pipeline import MiniBatchPipeline
    dg, hg = graph
    b, fan, seed, dim, cap = 256, (10, 5), 7, 64, 2000
    order = hg.train_nodes()[np.random.default_rng(0).permutation(hg.num_train())].astype(np.int32)
    nb = len(order) // b
    order = order[: nb * b]
    distinct = [cso.sample_batch(hg.row_offsets, hg.col_indices, order[i * b:(i + 1) * b].astype(np.int64), fan,
                                 seed, i)[2] for i in range(nb)]
    _, ref_codes = co.FifoEngine(cap, 0, 1).run(distinct + distinct[:3])
    feats = synthetic_features(hg.num_nodes, dim, seed=2, device_resident=(where == "hbm"))
    pipe = MiniBatchPipeline(dg, fan, b, torch.from_numpy(order).cuda(), seed,
                             CacheConfig(device_capacity=cap, feature_bytes_per_node=dim * 4), feats, rng="counter")
    pipe.capture()
    for i in range(nb):
        pipe.step()
        torch.cuda.synchronize()
        d = pipe.distinct().cpu().numpy()
        assert np.array_equal(d, distinct[i]), i
        assert np.array_equal(pipe.codes().cpu().numpy(), ref_codes[i]), i
        assert np.array_equal(pipe.rows().cpu().numpy(), fo.synthetic_features(d, dim, seed=2)), i
