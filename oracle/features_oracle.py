"""CPU oracle for feature retrieval (test oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference never materialises features (`gnnio/graph.py:3-6`); it only
counts bytes (`feature_bytes_per_node = 4 * feature_dim`, graph.py:41-43;
peer / host / remote bytes, cachesim.py:261-272). The retrieval contract the
build adds is `rows[i] = F[trace.batches[b][i]]`, byte-exact.

`synthetic_features` restates the counter hash the product's synthetic
generator uses, so tests can regenerate F on the CPU without storing it:
    key = (v << 20) | j,  z = splitmix64(key + seed * 0xD1B54A32D192ED03),
    F[v, j] = float32(((z >> 40) & 0xFFFFFF) * 2**-24 - 0.5)
"""

from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix(z):
    z = z.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = z ^ (z >> np.uint64(30))
        z = z * np.uint64(0xBF58476D1CE4E5B9)
        z = z ^ (z >> np.uint64(27))
        z = z * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def synthetic_features(ids, dim, seed=0):
    ids = np.asarray(ids, dtype=np.uint64)
    j = np.arange(dim, dtype=np.uint64)
    key = (ids[:, None] << np.uint64(20)) | j[None, :]
    with np.errstate(over="ignore"):
        z = key + np.uint64(seed) * np.uint64(0xD1B54A32D192ED03)
    z = _splitmix(z)
    return (((z >> np.uint64(40)) & np.uint64(0xFFFFFF)).astype(np.float64) / float(1 << 24) - 0.5).astype(np.float32)


def gather(features, ids):
    return np.asarray(features)[np.asarray(ids, dtype=np.int64)]
