"""CPU restatement of the counter-RNG sampler mode (test oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The counter-RNG mode (bgl_sample_hop_counter, csrc/sampler_counter.cu) is the
north_star's "uniform-fanout sampler with a counter-based RNG"; it has no
reference counterpart -- gnnio's sampler draws deg numpy doubles per parent
(sampler.py:65-94), which the replay mode reproduces bit for bit. This file
restates the counter mode exactly so the kernel can be checked bit for bit;
its statistical validity (every sample a neighbour, no duplicate per parent,
k = min(fanout, deg), uniform k-subsets) is checked in tests/test_gpu_counter.py.

  * Philox4x32-10 (Salmon et al., SC'11; Random123's round function, Weyl key
    schedule; known-answer vectors in tests);
  * key = hash of the batch stream's PCG64 (state, inc) that numpy's
    SeedSequence gives (seed, batch_seed) -- the device reads it from row 0 of
    the batch's jump table;
  * hop 0 (sub-warp per seed): k = min(fanout, deg); deg <= k -> all
    neighbours in adjacency order; else m = min(k, deg - k) slots draw
    uniform[0, deg) in rounds (slot s, round rho: Philox counter (q, h | rho
    << 8, s, 0), Lemire acceptance over its 4 outputs); a slot keeps its draw
    unless a slot already kept holds the value or a lower slot drew it in the
    same round; k <= deg/2 -> the kept values in slot order, else they are the
    excluded indices and the rest is emitted in adjacency order;
  * hops >= 1 (lane per parent, sample_hop_floyd): counter (q, h, block, 0);
    Floyd's algorithm: for j = deg-k .. deg-1: r = uniform[0, j], r = j if
    already chosen.
"""

from __future__ import annotations

import numpy as np

M32 = 0xFFFFFFFF


def philox4x32(ctr, key):
    c = [x & M32 for x in ctr]
    k0, k1 = key[0] & M32, key[1] & M32
    for r in range(10):
        if r:
            k0, k1 = (k0 + 0x9E3779B9) & M32, (k1 + 0xBB67AE85) & M32
        p0, p1 = 0xD2511F53 * c[0], 0xCD9E8D57 * c[2]
        c = [((p1 >> 32) ^ c[1] ^ k0) & M32, p1 & M32, ((p0 >> 32) ^ c[3] ^ k1) & M32, p0 & M32]
    return c


def stream_key(seed: int, batch_seed: int) -> tuple[int, int]:
    st = np.random.default_rng((seed, batch_seed)).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    a = (s >> 64) ^ (inc >> 64)
    b = (s & m) ^ (inc & m)
    k0 = ((a ^ (a >> 32)) & M32) ^ (b & M32)
    k1 = ((b >> 32) ^ (a >> 17)) & M32
    return k0, k1


class _Stream:
    def __init__(self, key, q, hop):
        self.key, self.q, self.hop, self.blk, self.buf = key, q, hop, 0, []

    def next(self):
        if not self.buf:
            self.buf = philox4x32([self.q, self.hop, self.blk, 0], self.key)
            self.blk += 1
        return self.buf.pop(0)

    def bounded(self, bound):
        m = self.next() * bound
        lo = m & M32
        if lo < bound:
            thr = ((1 << 32) - bound) % bound
            while lo < thr:
                m = self.next() * bound
                lo = m & M32
        return m >> 32


def sample_hop(row_offsets, col, parents, fanout, key, hop):
    out, pidx = [], []
    for q, p in enumerate(parents):
        off, deg = int(row_offsets[p]), int(row_offsets[p + 1] - row_offsets[p])
        k = min(fanout, deg)
        if deg <= k:
            out.extend(int(col[off + t]) for t in range(k))
        else:
            excl = 2 * k > deg
            m = deg - k if excl else k
            kept = [None] * m
            rho = 0
            thr = ((1 << 32) - deg) % deg
            while any(v is None for v in kept):
                draws = {}
                for sl in range(m):
                    if kept[sl] is None:
                        c = philox4x32([q, hop | (rho << 8), sl, 0], key)
                        for u in c:
                            mm = u * deg
                            if (mm & M32) >= thr:
                                draws[sl] = mm >> 32
                                break
                before = {v for v in kept if v is not None}
                for sl in sorted(draws):
                    v = draws[sl]
                    if v not in before and not any(draws[s2] == v for s2 in draws if s2 < sl):
                        kept[sl] = v
                rho += 1
            if excl:
                ex = set(kept)
                out.extend(int(col[off + t]) for t in range(deg) if t not in ex)
            else:
                out.extend(int(col[off + v]) for v in kept)
        pidx.extend([q] * k)
    return np.array(out, dtype=np.int64), np.array(pidx, dtype=np.int64)


def sample_hop_floyd(row_offsets, col, parents, fanout, key, hop):
    out, pidx = [], []
    for q, p in enumerate(parents):
        off, deg = int(row_offsets[p]), int(row_offsets[p + 1] - row_offsets[p])
        k = min(fanout, deg)
        if deg <= k:
            out.extend(int(col[off + t]) for t in range(k))
        else:
            rs, chosen = _Stream(key, q, hop), []
            for i in range(k):
                j = deg - k + i
                x = rs.bounded(j + 1)
                if x in chosen:
                    x = j
                chosen.append(x)
                out.append(int(col[off + x]))
        pidx.extend([q] * k)
    return np.array(out, dtype=np.int64), np.array(pidx, dtype=np.int64)


def sample_batch(row_offsets, col, seeds, fanouts, seed, batch_seed=0):
    key = stream_key(seed, batch_seed)
    parents = np.asarray(seeds, dtype=np.int64)
    frontiers, pidxs = [], []
    for h, f in enumerate(fanouts):
        hop_fn = sample_hop if h == 0 else sample_hop_floyd
        ids, pidx = hop_fn(row_offsets, col, parents, f, key, h)
        frontiers.append(ids)
        pidxs.append(pidx)
        parents = ids
    distinct = np.unique(np.concatenate([np.asarray(seeds, dtype=np.int64)] + frontiers))
    return frontiers, pidxs, distinct
