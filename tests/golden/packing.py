"""Flat (data, offsets) packing of ragged int arrays for the .npz fixtures."""

from __future__ import annotations

import numpy as np


def pack(arrays, dtype=np.int64):
    arrays = [np.asarray(a, dtype=dtype).ravel() for a in arrays]
    off = np.zeros(len(arrays) + 1, dtype=np.int64)
    off[1:] = np.cumsum([a.size for a in arrays])
    data = np.concatenate(arrays) if arrays else np.empty(0, dtype=dtype)
    return data.astype(dtype), off


def unpack(data, off):
    return [data[off[i]:off[i + 1]] for i in range(len(off) - 1)]


def put(store: dict, name: str, arrays, dtype=np.int64):
    store[name + "__data"], store[name + "__off"] = pack(arrays, dtype)


def get(npz, name: str):
    return unpack(npz[name + "__data"], npz[name + "__off"])
