"""Host-link read amplification of the miss gather under different row
layouts of the pinned feature store (C2): for batches of two epochs, the
device-missed rows (FIFO, 10% cache) are mapped through a layout (storage
position of node v) and the 64-B blocks their 400-B rows touch are counted.
Layouts: identity, full-graph BFS, reverse Cuthill-McKee, and first touch in
epoch 0 of the schedule (evaluated on epoch 1)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402
from scipy.sparse import csgraph  # noqa: E402

import bench  # noqa: E402
import paper_2112_08541_b200 as bgl  # noqa: E402

cfg = bench.CONFIGS["c2"]
n, b, rb, C = cfg["n"], cfg["b"], cfg["dim"] * 4, int(cfg["cache_frac"] * cfg["n"])
NB = int(os.environ.get("PROBE_BATCHES", 60))
dg, _, order, _ = bench.build_inputs(cfg, "hbm")
order = order.cpu().numpy()
nbl = (order.size + b - 1) // b
scfg = bgl.SamplingConfig(fanouts=cfg["fanouts"], seed=bench.RUN_SEED)


def trace(first):
    out = []
    for i in range(first, first + NB):
        s = order[(i % nbl) * b:(i % nbl + 1) * b]
        _, d = bgl.sample_batch(dg, s, scfg, batch_seed=i)
        out.append(d.astype(np.int64))
    return out


t0 = time.time()
ep0, ep1 = trace(0), trace(nbl)
print(f"traces {time.time() - t0:.1f}s, distinct/batch {np.mean([len(x) for x in ep0]):.0f}", flush=True)

# FIFO misses over epoch 0 then epoch 1 (closed form, cachesim.py:308-344)
resident = np.zeros(n, bool)
ring = np.full(C, -1, np.int64)
tail = 0
miss0, miss1 = [], []
for k, ids in enumerate(ep0 + ep1):
    m = ids[~resident[ids]]
    (miss0 if k < NB else miss1).append(m)
    M = m.size
    if M >= C:
        m = m[M - C:]
        tail = (tail + M - C) % C
        M = C
    pos = (tail + np.arange(M)) % C
    old = ring[pos]
    resident[old[old >= 0]] = False
    ring[pos] = m
    resident[m] = True
    tail = (tail + M) % C
print(f"misses/batch epoch0 {np.mean([x.size for x in miss0]):.0f} epoch1 {np.mean([x.size for x in miss1]):.0f}",
      flush=True)

hg = dg.to_host()
A = sp.csr_matrix((np.ones(hg.col_indices.size, np.int8), hg.col_indices, hg.row_offsets), shape=(n, n))


def bfs_layout():
    seen = np.zeros(n, bool)
    parts = []
    for r in np.argsort(-np.diff(hg.row_offsets), kind="stable"):
        if seen[r]:
            continue
        o = csgraph.breadth_first_order(A, r, directed=False, return_predecessors=False)
        seen[o] = True
        parts.append(o)
        if seen.all():
            break
    rest = np.flatnonzero(~seen)
    seq = np.concatenate(parts + [rest])
    pos = np.empty(n, np.int64)
    pos[seq] = np.arange(n)
    return pos


def first_touch_layout(tr):
    first = np.full(n, np.iinfo(np.int64).max, np.int64)
    for k, ids in enumerate(tr):
        f = first[ids]
        first[ids] = np.minimum(f, k)
    seq = np.lexsort((np.arange(n), first))
    pos = np.empty(n, np.int64)
    pos[seq] = np.arange(n)
    return pos


def cost(pos, misses, g=64):
    """(g-B blocks read) x g / (rows x 400) and mean contiguous-run length."""
    blocks = rows = runs = 0
    for m in misses:
        p = np.sort(pos[m])
        s, e = p * rb // g, (p * rb + rb - 1) // g
        blocks += int((e - s + 1).sum() - np.count_nonzero(s[1:] == e[:-1]))
        rows += p.size
        runs += 1 + int(np.count_nonzero(np.diff(p) != 1)) if p.size else 0
    return blocks * g / (rows * rb), rows / max(runs, 1)


layouts = {"identity": np.arange(n)}
t0 = time.time()
layouts["bfs"] = bfs_layout()
print(f"bfs {time.time() - t0:.1f}s", flush=True)
t0 = time.time()
rcm = csgraph.reverse_cuthill_mckee(A.astype(np.float32), symmetric_mode=True)
p_rcm = np.empty(n, np.int64)
p_rcm[rcm] = np.arange(n)
layouts["rcm"] = p_rcm
print(f"rcm {time.time() - t0:.1f}s", flush=True)
layouts["first_touch_epoch0"] = first_touch_layout(ep0)
layouts["first_touch_epoch1"] = first_touch_layout(ep1)     # oracle placement (upper bound)
rng = np.random.default_rng(0)
layouts["random"] = rng.permutation(n)
def pages(pos, misses, pg):
    """mean distinct pg-byte pages touched per batch by the miss rows."""
    return float(np.mean([np.unique(pos[m] * rb // pg).size for m in misses]))


for name, pos in layouts.items():
    print(f"{name:20s} pages/batch epoch1: 4K {pages(pos, miss1, 4096):.0f}  64K {pages(pos, miss1, 65536):.0f}  "
          f"2M {pages(pos, miss1, 2 << 20):.0f}", flush=True)
for name, pos in layouts.items():
    for g in (32, 64, 128):
        a0, r0 = cost(pos, miss0, g)
        a1, r1 = cost(pos, miss1, g)
        print(f"{name:20s} {g:3d}-B blocks  epoch0: amplification {a0:.3f} mean run {r0:.2f} rows | "
              f"epoch1: {a1:.3f}, {r1:.2f}", flush=True)
