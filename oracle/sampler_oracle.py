"""CPU restatement of the reference multi-hop sampler + dedup (test oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows `gnnio/sampler.py`:
  * batch stream  = `np.random.default_rng((cfg.seed, batch_seed))`  (sampler.py:61-62)
  * one hop       = per parent, `deg` uniform draws in CSR-segment order,
                    stable sort by (parent, priority), keep rank < fanout
                                                                     (sampler.py:65-94)
  * a batch       = hops chained, parents = previous samples, distinct =
                    sorted unique of seeds + all frontiers            (sampler.py:97-116)
  * an epoch      = batch rng keyed by batch index, partition accounting
                    (seed/request load, local/remote lookups)          (sampler.py:119-167)

Two formulations of a hop are given: `sample_hop` (vectorised, segment sort,
the reference's own formulation and the CPU baseline) and `sample_hop_topk`
(explicit per-parent "k smallest (m, t)" with 53-bit integer keys, the
formulation the CUDA kernel implements). Both are checked
against the reference's golden vectors.
"""

from __future__ import annotations

import numpy as np

TWO53 = float(1 << 53)


def batch_stream(seed: int, batch_seed: int) -> np.random.Generator:
    # sampler.py:61-62
    return np.random.default_rng((seed, batch_seed))


def _segments(row_offsets, parents):
    starts = row_offsets[parents]
    degs = row_offsets[parents + 1] - starts
    return starts, degs


def sample_hop(row_offsets, col, parents, fanout, rng):
    """(ids, parent_idx) for one hop; sampler.py:65-94."""
    parents = np.asarray(parents, dtype=np.int64)
    if parents.size == 0:
        return np.empty(0, np.int64), np.empty(0, np.int64)
    starts, degs = _segments(row_offsets, parents)
    total = int(degs.sum())
    if total == 0:
        return np.empty(0, np.int64), np.empty(0, np.int64)
    seg = np.repeat(np.arange(parents.size, dtype=np.int64), degs)
    seg_base = np.cumsum(degs) - degs
    t = np.arange(total, dtype=np.int64) - np.repeat(seg_base, degs)
    prio = rng.random(total)                      # sampler.py:90
    perm = np.lexsort((prio, seg))                # stable: ties keep t order (sampler.py:91)
    keep = t < fanout                             # t is the within-segment rank after sorting (sampler.py:92-93)
    sel = perm[keep]
    ids = np.asarray(col)[np.repeat(starts, degs)[sel] + t[sel]]
    return ids.astype(np.int64), seg[sel]


def sample_hop_topk(row_offsets, col, parents, fanout, rng):
    """Per-parent k-smallest restatement (small cases only; Python loop)."""
    parents = np.asarray(parents, dtype=np.int64)
    starts, degs = _segments(row_offsets, parents)
    total = int(degs.sum()) if parents.size else 0
    if total == 0:
        return np.empty(0, np.int64), np.empty(0, np.int64)
    m = (rng.random(total) * TWO53).astype(np.uint64)   # exact: u = m * 2**-53
    ids, pidx = [], []
    pos = 0
    for q in range(parents.size):
        d = int(degs[q])
        keys = sorted((int(m[pos + t]), t) for t in range(d))[: min(fanout, d)]
        ids.extend(int(col[starts[q] + t]) for _, t in keys)
        pidx.extend([q] * len(keys))
        pos += d
    return np.array(ids, np.int64), np.array(pidx, np.int64)


def sample_batch(row_offsets, col, seeds, fanouts, seed, batch_seed=0, hop=sample_hop):
    """(frontiers, parent_idx per hop, distinct, inverse) -- sampler.py:97-116.

    `inverse` is the relabel: rank of every key of concat(seeds, *frontiers)
    in `distinct` (np.unique(return_inverse)), the local-ID map the build
    defines."""
    seeds = np.asarray(seeds, dtype=np.int64)
    if seeds.size == 0:
        raise ValueError("seeds must be nonempty")
    rng = batch_stream(seed, batch_seed)
    frontiers, pidx = [], []
    parents = seeds
    for f in fanouts:
        ids, pi = hop(row_offsets, col, parents, int(f), rng)
        frontiers.append(ids)
        pidx.append(pi)
        parents = ids
    distinct, inverse = np.unique(np.concatenate([seeds] + frontiers), return_inverse=True)
    return frontiers, pidx, distinct, inverse


def simulate_epoch(row_offsets, col, part_of, k, batches, fanouts, seed):
    """Trace + comm accounting for one epoch -- sampler.py:119-167.

    Returns (trace batches, local, remote, seed_load, request_load)."""
    part_of = np.asarray(part_of, dtype=np.int64)
    local = remote = 0
    seed_load = np.zeros(k, np.int64)
    request_load = np.zeros(k, np.int64)
    trace = []
    for b, seeds in enumerate(batches):
        seeds = np.asarray(seeds, dtype=np.int64)
        rng = batch_stream(seed, b)
        seed_load += np.bincount(part_of[seeds], minlength=k)
        parents, origins = seeds, part_of[seeds]
        collected = [seeds]
        for f in fanouts:
            lp = part_of[parents]
            request_load += np.bincount(lp, minlength=k)
            n_local = int(np.count_nonzero(lp == origins))
            local += n_local
            remote += int(parents.size) - n_local
            ids, pi = sample_hop(row_offsets, col, parents, int(f), rng)
            origins = origins[pi]
            parents = ids
            collected.append(ids)
        trace.append(np.unique(np.concatenate(collected)))
    return trace, local, remote, seed_load, request_load
