"""CPU restatement of gnnio.graph.generate_power_law (test oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows `gnnio/graph.py:218-297` step by step, with every third-party
primitive it calls restated explicitly so the native generator
(`bgl_power_law_generate`, csrc/powerlaw.cu) can be checked draw by draw:

  * numpy 2.3 `Generator` over PCG64 (state taken from numpy's SeedSequence):
      random()       = (next64 >> 11) * 2**-53                  (graph.py:265, :278, :282)
      integers(h)    = Lemire's bounded draw on next_uint32 with
                       [0, h-1] and rejection threshold
                       (2**32 - h) % h; next_uint32 hands out the two
                       halves of one next64 (low half first, the high
                       half buffered in the bit generator)       (graph.py:266, :268, :285, :291)
      random(n)      = n x random()                             (graph.py:278)
      choice(n, size, replace=False):
                       n > 10000 and size > n // 50 -> tail shuffle of
                       arange(n) over i = n-1 .. n-size with bounded(i);
                       else Floyd's algorithm with bounded(j), j = n-size .. n-1
                                                                  (graph.py:295)
  * CPython 3.12 `set` insertion order of non-negative ints (hash = value):
    open addressing with 9 linear probes, then perturbed probing
    (i = 5i + 1 + perturb, perturb >>= 5); resize to the smallest power of
    two > 4 * used once fill * 5 >= mask * 3, re-inserting in table order.
    `for tgt in chosen` (graph.py:270) iterates the table in slot order.

`tests/golden/graph.npz` holds graphs produced by the reference itself
(`tests/golden/make_golden.py`); `tests/test_oracle_golden.py` pins this
restatement to them.
"""

from __future__ import annotations

import math

import numpy as np

M128 = (1 << 128) - 1
M64 = (1 << 64) - 1
MULT = 0x2360ED051FC65DA44385DF649FCCF645


class Pcg64Gen:
    """numpy Generator(PCG64) primitives used by the generator."""

    def __init__(self, state: int, inc: int, has_uint32: int = 0, uinteger: int = 0):
        self.s, self.inc, self.has32, self.u32 = state, inc, has_uint32, uinteger

    @classmethod
    def from_seed(cls, seed) -> "Pcg64Gen":
        st = np.random.default_rng(seed).bit_generator.state
        return cls(st["state"]["state"], st["state"]["inc"], st["has_uint32"], st["uinteger"])

    def next64(self) -> int:
        self.s = (self.s * MULT + self.inc) & M128
        x = (self.s >> 64) ^ (self.s & M64)
        rot = self.s >> 122
        return ((x >> rot) | (x << ((64 - rot) & 63))) & M64

    def next32(self) -> int:
        if self.has32:
            self.has32 = 0
            return self.u32
        v = self.next64()
        self.has32, self.u32 = 1, v >> 32
        return v & 0xFFFFFFFF

    def random(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)

    def bounded(self, rng: int) -> int:
        """Uniform integer in [0, rng] (rng < 2**32)."""
        if rng == 0:
            return 0
        if rng == 0xFFFFFFFF:
            return self.next32()
        excl = rng + 1
        m = self.next32() * excl
        left = m & 0xFFFFFFFF
        if left < excl:
            thr = (0xFFFFFFFF - rng) % excl
            while left < thr:
                m = self.next32() * excl
                left = m & 0xFFFFFFFF
        return m >> 32

    def integers(self, high: int) -> int:
        return self.bounded(high - 1)

    def choice_no_replace(self, n: int, size: int) -> list[int]:
        """The SET chosen by Generator.choice(n, size, replace=False) (its final
        shuffle only permutes the result and draws after every other use)."""
        if n > 10000 and size > n // 50:
            idx = list(range(n))
            for i in range(n - 1, max(n - size, 1) - 1, -1):
                j = self.bounded(i)
                idx[i], idx[j] = idx[j], idx[i]
            return idx[n - size:]
        chosen, out = set(), []
        for j in range(n - size, n):
            v = self.bounded(j)
            v = v if v not in chosen else j
            chosen.add(v)
            out.append(v)
        return out


class PySetOrder:
    """Insertion-ordered slot table of a CPython 3.12 set of non-negative ints."""

    LP = 9

    def __init__(self):
        self.mask, self.table, self.fill = 7, [None] * 8, 0

    def _insert_clean(self, key):
        perturb, i = key, key & self.mask
        while True:
            if self.table[i] is None:
                self.table[i] = key
                return
            if i + self.LP <= self.mask:
                for j in range(1, self.LP + 1):
                    if self.table[i + j] is None:
                        self.table[i + j] = key
                        return
            perturb >>= 5
            i = (i * 5 + 1 + perturb) & self.mask

    def add(self, key) -> None:
        mask, i, perturb = self.mask, key & self.mask, key
        while True:
            probes = self.LP if i + self.LP <= mask else 0
            e = i
            while True:
                if self.table[e] is None:
                    self.table[e] = key
                    self.fill += 1
                    if self.fill * 5 >= mask * 3:
                        minused = self.fill * 4 if self.fill <= 50000 else self.fill * 2
                        size = 8
                        while size <= minused:
                            size <<= 1
                        old, self.table, self.mask = self.table, [None] * size, size - 1
                        for k in old:
                            if k is not None:
                                self._insert_clean(k)
                    return
                if self.table[e] == key:
                    return
                if probes == 0:
                    break
                probes -= 1
                e += 1
            perturb >>= 5
            i = (i * 5 + 1 + perturb) & mask

    def __len__(self):
        return self.fill

    def __iter__(self):
        return (k for k in self.table if k is not None)


def power_law_edges(n: int, avg_degree: int, seed: int, train_fraction: float = 0.1, num_labels: int = 1,
                    cross_fraction: float = 0.05):
    """(edges int64 [E, 2] in generation order, labels int64 [n], sorted
    training IDs) exactly as generate_power_law draws them (graph.py:250-295)."""
    g = Pcg64Gen.from_seed(seed)
    m = max(1, int(round(avg_degree / 2)))                       # graph.py:251
    bounds = [i * n // num_labels for i in range(num_labels + 1)]
    labels = np.empty(n, dtype=np.int64)
    edges = []
    for c in range(num_labels):                                  # graph.py:256-274
        base, end = bounds[c], bounds[c + 1]
        labels[base:end] = c
        endpoints: list[int] = []
        for t in range(1, end - base):
            node, k = base + t, min(m, t)
            chosen = PySetOrder()
            while len(chosen) < k:
                if endpoints and g.random() < 0.9:
                    cand = endpoints[g.integers(len(endpoints))]
                else:
                    cand = base + g.integers(t)
                chosen.add(cand)
            for tgt in chosen:
                edges.append((node, tgt))
                endpoints.append(node)
                endpoints.append(tgt)
    if num_labels > 1 and cross_fraction > 0:                    # graph.py:276-291
        u = [g.random() for _ in range(n)]
        for v in (v for v in range(n) if u[v] < cross_fraction):
            c = int(labels[v])
            other = (c + (1 if g.random() < 0.5 else -1)) % num_labels
            lo, hi = bounds[other], bounds[other + 1]
            edges.append((v, lo + g.integers(hi - lo)))
        for c in range(num_labels):
            lo, hi = bounds[(c + 1) % num_labels], bounds[(c + 1) % num_labels + 1]
            edges.append((bounds[c], lo + g.integers(hi - lo)))
    num_train = int(math.floor(train_fraction * n))              # graph.py:293-295
    train = sorted(g.choice_no_replace(n, num_train))
    return np.array(edges, dtype=np.int64).reshape(-1, 2), labels, np.array(train, dtype=np.int64)


def csr_from_edges(edges: np.ndarray, n: int):
    """Sorted, deduplicated, symmetric CSR without self-loops (graph.py:88-107)."""
    e = edges[edges[:, 0] != edges[:, 1]]
    e = np.concatenate([e, e[:, ::-1]])
    keys = np.unique(e[:, 0] * n + e[:, 1])
    src, dst = keys // n, keys % n
    off = np.zeros(n + 1, dtype=np.int64)
    np.add.at(off, src + 1, 1)
    return np.cumsum(off), dst


# -- the same restatement in C (oracle/powerlaw_ref.c), for full-size shapes ----------

_CLIB = None


def _clib():
    """ctypes handle of oracle/_build/liboracle_graph.so (built by
    `make -C oracle`, which __graft_entry__.build() runs; built on first use
    when missing -- gcc is part of the image on the GPU box too)."""
    global _CLIB
    if _CLIB is None:
        import ctypes
        import os
        import subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        so = os.path.join(here, "_build", "liboracle_graph.so")
        if not os.path.exists(so):
            subprocess.run(["make", "-s", "-C", here], check=True)
        lib = ctypes.CDLL(so)
        i64, vp = ctypes.c_int64, ctypes.c_void_p
        lib.ref_power_law_edge_bound.restype = i64
        lib.ref_power_law_edge_bound.argtypes = [i64, i64, ctypes.c_int32]
        lib.ref_power_law_generate.restype = ctypes.c_int
        lib.ref_power_law_generate.argtypes = [i64, i64, ctypes.c_int32, ctypes.c_double, i64, vp, vp, vp, vp]
        lib.ref_csr_from_edges.restype = i64
        lib.ref_csr_from_edges.argtypes = [vp, i64, i64, vp, vp]
        _CLIB = lib
    return _CLIB


def generate_power_law_c(n: int, avg_degree: int, seed: int, train_fraction: float = 0.1, num_labels: int = 1,
                         cross_fraction: float = 0.05):
    """gnnio.graph.generate_power_law (graph.py:218-297) through the C
    restatement: (row_offsets int64 [n+1], col_indices int64 [E], train_mask
    bool [n], labels int64 [n]) -- the arrays the reference's Graph holds."""
    lib = _clib()
    m = max(1, int(round(avg_degree / 2)))                       # graph.py:251
    st = np.random.default_rng(seed).bit_generator.state
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    state = np.array([s >> 64, s & M64, inc >> 64, inc & M64, st["has_uint32"], st["uinteger"]], dtype=np.uint64)
    bound = int(lib.ref_power_law_edge_bound(n, m, num_labels))
    edges = np.empty((bound, 2), dtype=np.int32)
    ne = np.zeros(1, dtype=np.int64)
    train = np.zeros(n, dtype=np.uint8)
    rc = lib.ref_power_law_generate(n, m, num_labels, float(cross_fraction), int(math.floor(train_fraction * n)),
                                    state.ctypes.data, edges.ctypes.data, ne.ctypes.data, train.ctypes.data)
    if rc != 0:
        raise ValueError("generate_power_law_c: endpoint list beyond 2^32 entries (not restated)")
    E = int(ne[0])
    off = np.empty(n + 1, dtype=np.int64)
    col = np.empty(2 * E, dtype=np.int64)
    nnz = int(lib.ref_csr_from_edges(edges.ctypes.data, E, n, off.ctypes.data, col.ctypes.data))
    del edges
    col = col[:nnz].copy()
    bounds = np.array([i * n // num_labels for i in range(num_labels + 1)], dtype=np.int64)
    labels = (np.searchsorted(bounds, np.arange(n, dtype=np.int64), side="right") - 1).astype(np.int64)
    return off, col, train.astype(bool), labels
