"""Sampler parity on runs that mix hub parents (deg > 2048) with light ones,
for the kernels' rarely-taken paths (heavy-gap jumps in the segmented walk,
candidate-list overflow, the exact top-k fallback). Imported by
test_gpu_sampler_paths.py and run as a script under environment overrides
(BGL_SEG_CAP, BGL_RUNS_PER_SM, BGL_SAMPLER are read once per process)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import sampler_oracle as so  # noqa: E402


class G:
    def __init__(self, off, col):
        self.row_offsets = off
        self.col_indices = col
        self.num_nodes = len(off) - 1
        self.train_mask = np.zeros(self.num_nodes, bool)


def hub_graph(n=20000, hubs=(5, 6, 900, 4000, 4001), seed=3):
    """Chain + random edges, a few hubs of degree 2100-7000, 0..19 isolated."""
    rng = np.random.default_rng(seed)
    adj = [set() for _ in range(n)]
    for i, h in enumerate(hubs):
        for v in rng.choice(n, size=2100 + 1200 * i, replace=False):
            if v != h:
                adj[h].add(int(v)); adj[int(v)].add(h)
    for v in range(20, n - 1):
        if v % 7:
            adj[v].add(v + 1); adj[v + 1].add(v)
        for _ in range(2):
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
    return G(off, col), np.array(hubs)


FANOUTS = ((5, 5), (12, 3), (32,), (3, 3, 3))


def inputs(num_seeds=3000):
    g, hubs = hub_graph()
    rng = np.random.default_rng(7)
    seeds = rng.integers(0, g.num_nodes, num_seeds)
    seeds[::97] = hubs[np.arange(len(seeds[::97])) % len(hubs)]   # hubs inside every run
    return g, seeds


def expected(path):
    """Oracle frontiers + distinct for every fanout list (batch seed 3), saved to `path`."""
    g, seeds = inputs()
    out = {}
    for i, fanouts in enumerate(FANOUTS):
        fr_o, _, d_o, _ = so.sample_batch(g.row_offsets, g.col_indices, seeds, fanouts, 9, 3)
        for h, a in enumerate(fr_o):
            out[f"f{i}_h{h}"] = a
        out[f"f{i}_d"] = d_o
    np.savez(path, **out)


def check(path):
    import paper_2112_08541_b200 as bgl
    g, seeds = inputs()
    ref = np.load(path)
    for i, fanouts in enumerate(FANOUTS):
        fr, d = bgl.sample_batch(g, seeds, bgl.SamplingConfig(fanouts=fanouts, seed=9), batch_seed=3)
        for h, a in enumerate(fr):
            assert np.array_equal(a, ref[f"f{i}_h{h}"]), (fanouts, h)
        assert np.array_equal(d, ref[f"f{i}_d"]), fanouts


if __name__ == "__main__":
    check(sys.argv[1])
    print("ok")
