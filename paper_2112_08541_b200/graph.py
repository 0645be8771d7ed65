"""CSR graph container (mirror of gnnio.graph.Graph, graph.py:20-75), its
device-resident copy, the reference's power-law generator (bit-exact, native,
graph.py:218-297) and a GPU continuum-limit generator for the large configs.

The hot-path kernels consume `DeviceGraph`: int64 row offsets and int32
column indices in HBM (papers100M shape: 0.9 GB + 12.9 GB, resident in the
180 GB of one B200). Any object with `num_nodes`, `row_offsets`,
`col_indices` (and `train_mask` for ordering) is accepted, including the
reference's own `gnnio.graph.Graph`.
"""

from __future__ import annotations

import math
import weakref
from dataclasses import dataclass, field

import numpy as np
import torch


@dataclass
class Graph:
    """Immutable symmetric CSR graph (graph.py:20-75). `num_edges` counts
    directed adjacency entries; adjacency lists are sorted, duplicate-free,
    without self-loops."""

    num_nodes: int
    num_edges: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    labels: np.ndarray | None = None
    train_mask: np.ndarray = field(default=None)  # type: ignore[assignment]
    feature_dim: int = 128
    feature_bytes_per_node: int | None = None

    def __post_init__(self):
        if self.train_mask is None:
            self.train_mask = np.zeros(self.num_nodes, dtype=bool)
        if self.feature_bytes_per_node is None:
            self.feature_bytes_per_node = self.feature_dim * 4

    def degree(self, v: int) -> int:
        return int(self.row_offsets[v + 1] - self.row_offsets[v])

    def degrees(self) -> np.ndarray:
        return np.diff(self.row_offsets)

    def neighbors(self, v: int) -> np.ndarray:
        return self.col_indices[self.row_offsets[v]:self.row_offsets[v + 1]]

    def train_nodes(self) -> np.ndarray:
        return np.flatnonzero(self.train_mask)

    def num_train(self) -> int:
        return int(self.train_mask.sum())

    def validate(self) -> None:
        """Check the CSR invariants of graph.py:62-75; raises AssertionError
        on violation (vectorised: the same checks as the reference's per-node
        loop, with the same messages)."""
        off, col = np.asarray(self.row_offsets), np.asarray(self.col_indices)
        assert off[0] == 0 and off[-1] == self.num_edges
        assert len(off) == self.num_nodes + 1
        assert np.all(np.diff(off) >= 0)
        if self.num_edges:
            assert col.min() >= 0 and col.max() < self.num_nodes
            row = np.repeat(np.arange(self.num_nodes, dtype=np.int64), np.diff(off))
            same = row[1:] == row[:-1]
            bad = np.flatnonzero(same & (np.diff(col.astype(np.int64)) <= 0))
            assert bad.size == 0, f"adjacency of {int(row[bad[0] + 1]) if bad.size else -1} not sorted/deduped"
            loops = np.flatnonzero(col == row)
            assert loops.size == 0, f"self-loop at {int(row[loops[0]]) if loops.size else -1}"
        if self.labels is not None:
            assert np.all(self.labels[self.train_mask] >= 0)


class DeviceGraph:
    """CSR in HBM: indptr int64[n+1], indices int32[E]."""

    def __init__(self, indptr: torch.Tensor, indices: torch.Tensor, num_nodes: int,
                 train_mask: torch.Tensor | None = None, labels: torch.Tensor | None = None):
        assert indptr.is_cuda and indices.is_cuda
        assert indptr.dtype == torch.int64 and indices.dtype == torch.int32
        if num_nodes >= 2 ** 31:
            raise ValueError("node IDs must fit in int32")
        self.indptr = indptr.contiguous()
        self.indices = indices.contiguous()
        self.num_nodes = int(num_nodes)
        self.num_edges = int(indices.numel())
        self.train_mask = train_mask
        self.labels = labels
        deg = self.indptr[1:] - self.indptr[:-1]
        self.max_degree = int(deg.max().item()) if num_nodes > 0 else 0

    @classmethod
    def from_arrays(cls, row_offsets, col_indices, num_nodes, device=None, train_mask=None):
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        ip = torch.as_tensor(np.asarray(row_offsets, dtype=np.int64)).to(dev)
        ix = torch.as_tensor(np.asarray(col_indices).astype(np.int32, copy=False)).to(dev)
        tm = None if train_mask is None else torch.as_tensor(np.asarray(train_mask, dtype=bool)).to(dev)
        return cls(ip, ix, num_nodes, tm)

    def to_host(self) -> Graph:
        ro = self.indptr.cpu().numpy()
        ci = self.indices.cpu().numpy().astype(np.int64)      # the reference's dtype (graph.py:31)
        tm = self.train_mask.cpu().numpy() if self.train_mask is not None else None
        lb = self.labels.cpu().numpy() if self.labels is not None else None
        return Graph(self.num_nodes, int(ci.size), ro, ci, labels=lb, train_mask=tm)


_DEVICE_GRAPHS: dict[int, tuple[weakref.ref | None, DeviceGraph]] = {}


def device_graph(g) -> DeviceGraph:
    """Device copy of a host graph, uploaded once per graph object."""
    if isinstance(g, DeviceGraph):
        return g
    key = id(g)
    hit = _DEVICE_GRAPHS.get(key)
    if hit is not None and (hit[0] is None or hit[0]() is g):
        dg = hit[1]
        if dg.indptr.device.index == torch.cuda.current_device():
            return dg
    dg = DeviceGraph.from_arrays(g.row_offsets, g.col_indices, g.num_nodes,
                                 train_mask=getattr(g, "train_mask", None))
    try:
        ref = weakref.ref(g, lambda _r, k=key: _DEVICE_GRAPHS.pop(k, None))
    except TypeError:
        ref = None
    _DEVICE_GRAPHS[key] = (ref, dg)
    return dg


# ----------------------------------------------------------------------------- generator

def _check_generator_args(n, avg_degree, train_fraction, num_labels):
    # graph.py:239-248 (same messages)
    if n < 2:
        raise ValueError("n must be >= 2")
    if avg_degree < 1:
        raise ValueError("avg_degree must be >= 1")
    if avg_degree >= n:
        raise ValueError("avg_degree must be < n")
    if not 0 < train_fraction <= 1:
        raise ValueError("train_fraction must be in (0, 1]")
    if num_labels < 1 or num_labels > n:
        raise ValueError("num_labels must be in [1, n]")


def power_law_edges(n: int, avg_degree: int, seed: int, train_fraction: float = 0.1, num_labels: int = 1,
                    cross_fraction: float = 0.05):
    """The reference generator's raw output, bit-exact: (edges int32 [E, 2] in
    generation order, train_mask bool [n], labels int64 [n]). The sequential
    preferential-attachment process runs natively (bgl_power_law_generate);
    numpy supplies only the SeedSequence hash of `seed` (graph.py:250)."""
    from . import _lib
    _check_generator_args(n, avg_degree, train_fraction, num_labels)
    lib = _lib.load(require_cuda=False)
    m = max(1, int(round(avg_degree / 2)))                  # graph.py:251
    st = np.random.default_rng(seed).bit_generator.state    # graph.py:250
    s, inc = st["state"]["state"], st["state"]["inc"]
    mask = (1 << 64) - 1
    ps = np.array([s >> 64, s & mask, inc >> 64, inc & mask, st["has_uint32"], st["uinteger"]], dtype=np.uint64)
    bound = int(lib.bgl_power_law_edge_bound(n, m, num_labels))
    edges = np.empty((bound, 2), dtype=np.int32)
    ne = _lib.c_i64()
    train = np.empty(n, dtype=np.uint8)
    _lib.check(lib.bgl_power_law_generate(n, m, num_labels, float(cross_fraction), int(math.floor(train_fraction * n)),
                                          ps.ctypes.data, edges.ctypes.data, bound, _lib.ctypes.byref(ne),
                                          train.ctypes.data))
    bounds = [i * n // num_labels for i in range(num_labels + 1)]
    labels = np.repeat(np.arange(num_labels, dtype=np.int64), np.diff(bounds))
    return edges[: ne.value], train.astype(bool), labels


def csr_from_edges_device(edges: np.ndarray, n: int, dev=None, max_keys: int = 1 << 29) -> tuple[torch.Tensor, torch.Tensor]:
    """Sorted, deduplicated, symmetric CSR without self-loops on the device
    (csr_from_edges, graph.py:88-107): (indptr int64 [n+1], indices int32).
    Large edge lists (CUB sorts < 2^31 keys; papers100M has 3.1B directed
    keys) are keyed and deduplicated per source-node range."""
    dev = torch.device("cuda", torch.cuda.current_device()) if dev is None else torch.device(dev)
    E = int(edges.shape[0])
    limit = max(2, int(max_keys))          # directed keys per pass (both directions of <= limit/2 edges)
    nchunks = max(1, -(-2 * E // limit))
    counts = torch.zeros(n, dtype=torch.int64, device=dev)
    cols = []
    bounds = [c * n // nchunks for c in range(nchunks + 1)]
    for c in range(nchunks):
        lo, hi = bounds[c], bounds[c + 1]
        parts = []
        for e0 in range(0, E, limit // 2):    # stream the host edge list through the device
            e = torch.from_numpy(np.ascontiguousarray(edges[e0:e0 + limit // 2])).to(dev)
            src, dst = e[:, 0].to(torch.int64), e[:, 1].to(torch.int64)
            del e
            keep = src != dst
            src, dst = src[keep], dst[keep]
            for a, b in ((src, dst), (dst, src)):
                m = (a >= lo) & (a < hi)
                if nchunks == 1:
                    parts.append(a * n + b)
                else:
                    parts.append(a[m] * n + b[m])
            del src, dst, keep
        key = torch.unique(torch.cat(parts))
        del parts
        row = key // n
        cols.append((key - row * n).to(torch.int32))
        counts += torch.bincount(row, minlength=n)
        del key, row
    indptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    indptr[1:] = torch.cumsum(counts, 0)
    return indptr, torch.cat(cols) if len(cols) > 1 else cols[0]


def generate_power_law_exact_device(n: int, avg_degree: int, seed: int, train_fraction: float = 0.1,
                                    num_labels: int = 1, cross_fraction: float = 0.05, device=None) -> DeviceGraph:
    """gnnio.graph.generate_power_law(...) (graph.py:218-297), bit-identical,
    built straight into HBM: native edge process + device CSR."""
    edges, train, labels = power_law_edges(n, avg_degree, seed, train_fraction, num_labels, cross_fraction)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    indptr, col = csr_from_edges_device(edges, n, dev)
    del edges
    return DeviceGraph(indptr, col, n, train_mask=torch.from_numpy(train).to(dev),
                       labels=torch.from_numpy(labels).to(dev))


def generate_power_law(n: int, avg_degree: int, seed: int, train_fraction: float = 0.1, num_labels: int = 1,
                       cross_fraction: float = 0.05) -> Graph:
    """Drop-in for gnnio.graph.generate_power_law (graph.py:218-297): the same
    host `Graph`, bit-identical (tests/golden/graphgen.npz), from the native
    generator with the CSR built on the device."""
    dg = generate_power_law_exact_device(n, avg_degree, seed, train_fraction, num_labels, cross_fraction)
    return dg.to_host()


def generate_power_law_device(n: int, avg_degree: int, seed: int, train_fraction: float = 0.1,
                              num_labels: int = 1, cross_fraction: float = 0.05,
                              device=None) -> DeviceGraph:
    """Same graph MODEL as generate_power_law, generated entirely on the GPU in
    its continuum limit (power_law_csr) -- NOT bit-exact; for shapes where the
    sequential exact process is too long (papers100M: 1.55B edges)."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    indptr, col, train_mask, comm = power_law_csr(n, avg_degree, seed, train_fraction, num_labels,
                                                  cross_fraction, dev)
    return DeviceGraph(indptr, col, n, train_mask=train_mask, labels=comm)


PREF_FRACTION = 0.9   # degree-proportional share of the picks (graph.py:257)
CORE_FACTOR = 0.5     # BA core size t0 = CORE_FACTOR * m (max degree ~ sqrt(2 m N_community))


def power_law_csr(n: int, avg_degree: int, seed: int, train_fraction: float, num_labels: int,
                  cross_fraction: float, dev):
    """Power-law graph with planted communities, built on the GPU.

    Same shape model as gnnio.graph.generate_power_law (graph.py:218-297):
    `num_labels` contiguous ID-range communities, each grown by preferential
    attachment with m = round(avg_degree / 2) edges per new node (90% degree-
    proportional, 10% uniform), `cross_fraction` of nodes with one edge into a
    ring-adjacent community, one bridge per ring step, floor(train_fraction *
    n) training nodes. The reference's sequential endpoint-list process is
    replaced by its continuum limit -- a node t attaches to t' in [t0, t) with
    density proportional to t'^(-1/2), the Barabasi-Albert attachment kernel
    (degree of t' ~ m sqrt(t / t')) -- so the whole graph is a few sorts on the
    device. Calibrated against the reference generator: at the C2 shape (n =
    2.4M, avg_degree 51, 47 labels) max degree 1578 vs 1733 and E[d^2]/E[d]
    106 vs 112; at C1 (100K, 20, 64) 194 vs 221 and 31.8 vs 36. It is a
    benchmark input generator, not bit-exact with the reference's.
    """
    if n < 2 or avg_degree < 1 or avg_degree >= n:
        raise ValueError("need n >= 2 and 1 <= avg_degree < n")
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed))
    m = max(1, int(round(avg_degree / 2)))
    L = num_labels
    bounds = torch.tensor([i * n // L for i in range(L + 1)], dtype=torch.int64, device=dev)
    node = torch.arange(n, dtype=torch.int64, device=dev)
    comm = torch.searchsorted(bounds, node, right=True) - 1
    base = bounds[comm]
    t = node - base
    srcs, dsts = [], []
    chunk = max(1, (1 << 27) // m)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        tt = t[lo:hi].unsqueeze(1).expand(-1, m)
        u = torch.rand(tt.shape, generator=gen, device=dev, dtype=torch.float64)
        pref = torch.rand(tt.shape, generator=gen, device=dev) < PREF_FRACTION
        tf = tt.to(torch.float64)
        # BA continuum: node t' (>= t0) has degree ~ m sqrt(t / t'), so a new
        # node t picks t' with density ~ t'^(-1/2) on [t0, t):
        # t' = (sqrt(t0) + U (sqrt(t) - sqrt(t0)))^2
        t0 = torch.minimum(torch.full_like(tf, CORE_FACTOR * m), tf)
        st0 = torch.sqrt(t0)
        prefpick = torch.floor((st0 + u * (torch.sqrt(tf) - st0)) ** 2)
        tgt = torch.where(pref, prefpick, torch.floor(tf * u)).to(torch.int64)
        tgt = torch.minimum(tgt, (tt - 1).clamp_min(0))
        valid = torch.arange(m, device=dev).unsqueeze(0) < torch.minimum(tt, torch.full_like(tt, m))
        s = node[lo:hi].unsqueeze(1).expand(-1, m)[valid]
        d = (base[lo:hi].unsqueeze(1) + tgt)[valid]
        srcs.append(s)
        dsts.append(d)
    if L > 1 and cross_fraction > 0:
        pick = torch.rand(n, generator=gen, device=dev) < cross_fraction
        v = node[pick]
        side = torch.where(torch.rand(v.numel(), generator=gen, device=dev) < 0.5, 1, -1)
        other = (comm[pick] + side) % L
        lo, hi = bounds[other], bounds[other + 1]
        partner = lo + (torch.rand(v.numel(), generator=gen, device=dev, dtype=torch.float64)
                        * (hi - lo).to(torch.float64)).to(torch.int64)
        srcs.append(v)
        dsts.append(partner)
        c = torch.arange(L, device=dev)
        nx = (c + 1) % L
        lo, hi = bounds[nx], bounds[nx + 1]
        partner = lo + (torch.rand(L, generator=gen, device=dev, dtype=torch.float64)
                        * (hi - lo).to(torch.float64)).to(torch.int64)
        srcs.append(bounds[:-1])
        dsts.append(partner)
    src = torch.cat(srcs)
    dst = torch.cat(dsts)
    del srcs, dsts
    keep = src != dst
    src, dst = src[keep], dst[keep]
    key = torch.cat([src * n + dst, dst * n + src])
    del src, dst, keep
    # sorted, deduplicated (symmetric CSR, graph.py:88-107); CUB sorts < 2^31
    # items, so large graphs are deduplicated per source-node range
    limit = 1 << 30
    if key.numel() <= limit:
        key = torch.unique(key)
    else:
        pieces = []
        nchunks = (key.numel() + limit - 1) // limit * 2
        for c in range(nchunks):
            lo, hi = c * n // nchunks, (c + 1) * n // nchunks
            pieces.append(torch.unique(key[(key >= lo * n) & (key < hi * n)]))
        del key
        key = torch.cat(pieces)
        del pieces
    row = key // n
    col = (key - row * n).to(torch.int32)
    del key
    counts = torch.bincount(row, minlength=n)
    del row
    indptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    indptr[1:] = torch.cumsum(counts, 0)
    num_train = int(math.floor(train_fraction * n))
    train_mask = torch.zeros(n, dtype=torch.bool, device=dev)
    train_mask[torch.randperm(n, generator=gen, device=dev)[:num_train]] = True
    return indptr, col, train_mask, comm
