"""CPU restatement of the reference proximity-aware ordering (test oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows `gnnio/ordering.py`:
  * S contiguous shards of the ascending training IDs; one rng for the call;
    per restart root = pending[rng.integers(len(pending))]; level-synchronous
    BFS over the full graph emitting not-yet-emitted shard members in
    frontier order; next frontier = unvisited neighbours in parent order,
    first occurrence kept; `visited` persists across restarts of a shard
                                                             (ordering.py:57-116)
  * rotation by default_rng(seed).integers(len)              (ordering.py:119-126)
  * round-robin interleave into batches of b, closed form
    pos(i, r) = sum_j min(L_j, r) + #{j < i : L_j > r}       (ordering.py:129-151)
  * proximity_schedule = shards -> shift(seed*1000003+i) -> interleave
                                                             (ordering.py:192-196)
  * random schedule = permutation of the training IDs sliced by b
                                                             (ordering.py:199-207)
"""

from __future__ import annotations

import numpy as np


def bfs_sequences(row_offsets, col, train_mask, S, seed):
    train = np.flatnonzero(train_mask)
    if train.size == 0:
        raise ValueError("training set is empty")
    if S < 1:
        raise ValueError("S must be >= 1")
    if S > train.size:
        raise ValueError(f"S={S} exceeds training-set size {train.size}")
    n = len(row_offsets) - 1
    rng = np.random.default_rng(seed)
    out = []
    for s in range(S):
        shard = train[s * train.size // S:(s + 1) * train.size // S]
        member = np.zeros(n, bool)
        member[shard] = True
        done = np.zeros(n, bool)      # emitted
        seen = np.zeros(n, bool)      # visited
        pieces = []
        left = shard.size
        while left > 0:
            pend = shard[~done[shard]]
            root = int(pend[rng.integers(pend.size)])
            front = np.array([root], np.int64)
            seen[root] = True
            while front.size and left > 0:
                em = front[member[front] & ~done[front]]
                if em.size:
                    done[em] = True
                    left -= em.size
                    pieces.append(em)
                lo = row_offsets[front]
                cnt = row_offsets[front + 1] - lo
                tot = int(cnt.sum())
                if tot == 0:
                    break
                base = np.cumsum(cnt) - cnt
                cand = col[np.repeat(lo - base, cnt) + np.arange(tot)]
                cand = cand[~seen[cand]]
                if cand.size == 0:
                    break
                _, first = np.unique(cand, return_index=True)
                front = cand[np.sort(first)].astype(np.int64)
                seen[front] = True
        out.append(np.concatenate(pieces) if pieces else np.empty(0, np.int64))
    return out


def rotate(seq, seed):
    if len(seq) == 0:
        raise ValueError("sequence is empty")
    r = int(np.random.default_rng(seed).integers(len(seq)))
    return np.concatenate([seq[r:], seq[:r]])


def interleave(seqs, b):
    """Closed-form round-robin; returns the flat order and batch list."""
    if b < 1:
        raise ValueError("batch size must be >= 1")
    lens = np.array([len(s) for s in seqs], dtype=np.int64)
    total = int(lens.sum())
    flat = np.empty(total, dtype=np.int64)
    for i, s in enumerate(seqs):
        r = np.arange(lens[i])
        pos = np.minimum(lens[None, :], r[:, None]).sum(axis=1) + (lens[None, :i] > r[:, None]).sum(axis=1)
        flat[pos] = s
    return flat, [flat[i:i + b] for i in range(0, total, b)]


def proximity_schedule(row_offsets, col, train_mask, S, b, seed):
    seqs = bfs_sequences(row_offsets, col, train_mask, S, seed)
    shifted = [rotate(s, seed * 1000003 + i) if len(s) else s for i, s in enumerate(seqs)]
    return interleave(shifted, b)[1]


def random_schedule(train_mask, b, seed):
    if b < 1:
        raise ValueError("batch size must be >= 1")
    perm = np.random.default_rng(seed).permutation(np.flatnonzero(train_mask))
    return [perm[i:i + b] for i in range(0, perm.size, b)]
