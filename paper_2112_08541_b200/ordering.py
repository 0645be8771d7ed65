"""Proximity-aware mini-batch ordering on the B200 (drop-in for gnnio.ordering).

Public surface of the reference (`gnnio/ordering.py`): `BatchSchedule`
(:20-32), `generate_bfs_sequences` (:57-116), `random_shift` (:119-126),
`form_batches` (:129-151), `proximity_schedule` (:192-196),
`random_shuffle_schedule` (:199-207), `save_schedule` / `load_schedule`
(:237-261). The BFS levels and the interleave run on the device
(`bgl_bfs_level`, `bgl_select_pending`, `bgl_interleave`); the host keeps the
numpy rng -- one `integers` draw per BFS restart and one per rotation, the
"few scalars" of SURVEY.md §8 a15/a16 -- so the schedule is bit-exact.
Random shuffling (a permutation of at most a few million IDs) stays in host
numpy, as the reference's own single call.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .graph import DeviceGraph, device_graph


@dataclass
class BatchSchedule:
    batches: list[np.ndarray]
    batch_size: int
    policy: str

    def all_nodes(self) -> np.ndarray:
        if not self.batches:
            return np.empty(0, dtype=np.int64)
        return np.concatenate(self.batches)

    def num_nodes(self) -> int:
        return sum(len(b) for b in self.batches)


class BfsEngine:
    """Device buffers for level-synchronous BFS over one graph."""

    def __init__(self, dg: DeviceGraph):
        self.dg = dg
        n = dg.num_nodes
        dev = dg.indptr.device
        self.flags = torch.zeros(n, dtype=torch.uint8, device=dev)
        self.best = torch.full((n,), 2 ** 63 - 1, dtype=torch.int64, device=dev)
        self.front = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(2)]
        self.scal = torch.zeros(4, dtype=torch.int64, device=dev)   # n_front[2], seq_len, remaining
        self.ws = torch.empty(int(_lib.load().bgl_bfs_workspace(n)), dtype=torch.uint8, device=dev)

    def shard_sequence(self, shard: torch.Tensor, rng: np.random.Generator) -> torch.Tensor:
        """BFS first-visit order of one shard (ordering.py:79-114)."""
        lib = _lib.load()
        st = _lib.stream_ptr()
        dg = self.dg
        n = dg.num_nodes
        L = int(shard.numel())
        seq = torch.empty(max(L, 1), dtype=torch.int32, device=shard.device)
        self.flags.zero_()
        self.flags[shard.long()] = 1
        self.scal.zero_()
        self.scal[3] = L
        sp = self.scal.data_ptr()
        n_front = [sp, sp + 8]
        seq_len, remaining = sp + 16, sp + 24
        remaining_h = L
        while remaining_h > 0:
            r = int(rng.integers(remaining_h))        # len(pending) == remaining (ordering.py:89-90)
            cur = 0
            _lib.check(lib.bgl_select_pending(shard.data_ptr(), L, self.flags.data_ptr(), r,
                                              self.front[cur].data_ptr(), n_front[cur], self.ws.data_ptr(), n, st))
            front_h = 1
            while True:
                _lib.check(lib.bgl_bfs_level(dg.indptr.data_ptr(), dg.indices.data_ptr(), n, self.flags.data_ptr(),
                                             self.front[cur].data_ptr(), n_front[cur], front_h, seq.data_ptr(),
                                             seq_len, self.front[1 - cur].data_ptr(), n_front[1 - cur], n,
                                             self.best.data_ptr(), self.ws.data_ptr(), remaining, st))
                h = self.scal.cpu().tolist()
                remaining_h = int(h[3])
                front_h = int(h[1 - cur])
                if remaining_h == 0 or front_h == 0:
                    break
                cur = 1 - cur
        return seq[:L]


_ENGINES: dict = {}


def _engine(dg: DeviceGraph) -> BfsEngine:
    e = _ENGINES.get(id(dg))
    if e is None or e.dg is not dg:
        _ENGINES.clear()
        e = BfsEngine(dg)
        _ENGINES[id(dg)] = e
    return e


def _train_ids(g) -> np.ndarray:
    tm = g.train_mask
    if isinstance(tm, torch.Tensor):
        return torch.nonzero(tm).flatten().cpu().numpy()
    return np.flatnonzero(np.asarray(tm))


def generate_bfs_sequences_device(g, S: int, seed: int = 0) -> list[torch.Tensor]:
    train = _train_ids(g)
    if len(train) == 0:
        raise ValueError("training set is empty")
    if S < 1:
        raise ValueError("S must be >= 1")
    if S > len(train):
        raise ValueError(f"S={S} exceeds training-set size {len(train)}")
    dg = device_graph(g)
    eng = _engine(dg)
    rng = np.random.default_rng(seed)                     # one rng for the call (ordering.py:74)
    train_dev = torch.from_numpy(train.astype(np.int32)).cuda()
    bounds = [i * len(train) // S for i in range(S + 1)]  # contiguous shards (ordering.py:75, 80)
    return [eng.shard_sequence(train_dev[bounds[s]:bounds[s + 1]], rng) for s in range(S)]


def generate_bfs_sequences(g, S: int, seed: int = 0) -> list[np.ndarray]:
    """Each shard's members in BFS first-visit order (ordering.py:57-116)."""
    return [s.cpu().numpy().astype(np.int64) for s in generate_bfs_sequences_device(g, S, seed)]


def random_shift(seq: np.ndarray, seed: int = 0) -> np.ndarray:
    """Rotate by a uniform offset (ordering.py:119-126)."""
    if len(seq) == 0:
        raise ValueError("sequence is empty")
    r = int(np.random.default_rng(seed).integers(len(seq)))
    return np.roll(np.asarray(seq), -r)


def _interleave_device(seqs: list[torch.Tensor], shifts: list[int]) -> torch.Tensor:
    lens = [int(s.numel()) for s in seqs]
    total = sum(lens)
    out = torch.empty(max(total, 1), dtype=torch.int32, device="cuda")
    if total == 0:
        return out[:0]
    cat = torch.cat([s.to(device="cuda", dtype=torch.int32) for s in seqs])
    off = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int64, device="cuda")
    sh = torch.tensor(shifts, dtype=torch.int64, device="cuda")
    _lib.call("bgl_interleave", cat.data_ptr(), off.data_ptr(), sh.data_ptr(), len(seqs), total, out.data_ptr(),
              _lib.stream_ptr())
    return out[:total]


def _slice(flat: np.ndarray, b: int) -> list[np.ndarray]:
    return [flat[i:i + b] for i in range(0, len(flat), b)]


def form_batches(seqs: list[np.ndarray], b: int, policy: str = "proximity") -> BatchSchedule:
    """Round-robin one node per live sequence per turn, sliced into batches of
    b (ordering.py:129-151); closed form on the device."""
    if b < 1:
        raise ValueError("batch size must be >= 1")
    if not seqs or sum(len(s) for s in seqs) == 0:
        return BatchSchedule(batches=[], batch_size=b, policy=policy)
    dev = [torch.as_tensor(np.asarray(s, dtype=np.int64)).to(torch.int32) for s in seqs]
    flat = _interleave_device(dev, [0] * len(seqs)).cpu().numpy().astype(np.int64)
    return BatchSchedule(batches=_slice(flat, b), batch_size=b, policy=policy)


def proximity_schedule_device(g, S: int, b: int, seed: int = 0) -> tuple[torch.Tensor, int]:
    """Device-resident flat proximity order (batches are consecutive b-slices)."""
    if b < 1:
        raise ValueError("batch size must be >= 1")
    seqs = generate_bfs_sequences_device(g, S, seed=seed)
    shifts = []
    for i, s in enumerate(seqs):
        L = int(s.numel())
        # random_shift(seq, seed*1000003+i), skipped for empty sequences (ordering.py:195)
        shifts.append(int(np.random.default_rng(seed * 1000003 + i).integers(L)) if L else 0)
    return _interleave_device(seqs, shifts), b


def proximity_schedule(g, S: int, b: int, seed: int = 0) -> BatchSchedule:
    """Shifted BFS sequences consumed round-robin (ordering.py:192-196)."""
    flat, b = proximity_schedule_device(g, S, b, seed)
    return BatchSchedule(batches=_slice(flat.cpu().numpy().astype(np.int64), b), batch_size=b,
                         policy=f"proximity-S{S}")


def random_shuffle_schedule(g, b: int, seed: int = 0) -> BatchSchedule:
    """Uniform permutation of the training set sliced into batches
    (ordering.py:199-207)."""
    if b < 1:
        raise ValueError("batch size must be >= 1")
    perm = np.random.default_rng(seed).permutation(_train_ids(g))
    return BatchSchedule(batches=_slice(perm, b), batch_size=b, policy="random")


# ----------------------------------------------------------------------------- shuffling error

@dataclass
class ShufflingErrorReport:
    """ordering.py:35-46."""

    epsilon: float
    threshold: float
    num_sequences: int
    per_batch_tv: np.ndarray
    max_tv: float = 0.0
    threshold_met: bool = True

    def __post_init__(self):
        if len(self.per_batch_tv):
            self.max_tv = float(np.max(self.per_batch_tv))


def shuffling_error_threshold(b: int, M: int, n: int) -> float:
    """Convergence-safe bound sqrt(b*M)/n (ordering.py:49-51)."""
    import math
    return math.sqrt(b * M) / n


def _device_labels(labels) -> tuple[torch.Tensor, int]:
    if isinstance(labels, torch.Tensor):
        lab = labels.to(device="cuda", dtype=torch.int32)
        return lab, int(lab.max().item()) + 1 if lab.numel() else 1
    lab = np.asarray(labels)
    return torch.from_numpy(lab.astype(np.int32)).cuda(), int(lab.max()) + 1 if lab.size else 1


def batch_tv_device(labels_dev: torch.Tensor, num_classes: int, order: torch.Tensor,
                    batch_off: torch.Tensor) -> torch.Tensor:
    """Per-batch TV distances (fp64, device) of a flat schedule (bgl_shuffling_tv)."""
    nb = int(batch_off.numel()) - 1
    total = int(order.numel())
    tv = torch.empty(max(nb, 1), dtype=torch.float64, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws = torch.empty(int(_lib.load().bgl_shuffling_workspace(num_classes)), dtype=torch.uint8, device="cuda")
    _lib.call("bgl_shuffling_tv", labels_dev.data_ptr(), order.data_ptr(), total, batch_off.data_ptr(), nb,
              num_classes, ws.data_ptr(), tv.data_ptr(), bad.data_ptr(), _lib.stream_ptr())
    if int(bad.item()):
        raise ValueError("scheduled node without a label")
    return tv[:nb]


def _epsilon(tvs: np.ndarray, lens: np.ndarray, batch_size: int) -> float:
    full = lens == batch_size
    return float(tvs[full].mean()) if full.any() else float(tvs.mean())


def shuffling_error(schedule: BatchSchedule, labels, threshold: float = 0.0,
                    num_sequences: int = 1) -> ShufflingErrorReport:
    """Per-batch total-variation distance of label frequencies vs the whole
    schedule's; epsilon = mean over full-size batches (ordering.py:157-186)."""
    lens = np.array([len(b) for b in schedule.batches], dtype=np.int64)
    lab, ncls = _device_labels(labels)
    order = torch.from_numpy(schedule.all_nodes().astype(np.int32)).cuda()
    off = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)).cuda()
    tvs = batch_tv_device(lab, ncls, order, off).cpu().numpy()
    eps = _epsilon(tvs, lens, schedule.batch_size)
    return ShufflingErrorReport(epsilon=eps, threshold=threshold, num_sequences=num_sequences, per_batch_tv=tvs,
                                threshold_met=eps <= threshold if threshold > 0 else True)


def select_num_sequences(g, b: int, M: int, S_max: int, seed: int = 0) -> tuple[int, ShufflingErrorReport]:
    """Smallest S in [1, S_max] whose shifted-BFS schedule keeps the shuffling
    error within sqrt(b*M)/n (ordering.py:210-231); every candidate schedule
    and its error are computed on the device."""
    if S_max < 1:
        raise ValueError("S_max must be >= 1")
    labels = getattr(g, "labels", None)
    if labels is None:
        raise ValueError("graph has no labels")
    n = len(_train_ids(g))
    threshold = shuffling_error_threshold(b, M, n)
    lab, ncls = _device_labels(labels)
    last = None
    for S in range(1, S_max + 1):
        flat, _ = proximity_schedule_device(g, S, b, seed=seed)
        total = int(flat.numel())
        lens = np.array([min(b, total - i) for i in range(0, total, b)], dtype=np.int64)
        off = torch.arange(0, total + b, b, dtype=torch.int64, device="cuda").clamp_max(total)[: len(lens) + 1]
        tvs = batch_tv_device(lab, ncls, flat, off).cpu().numpy()
        eps = _epsilon(tvs, lens, b)
        last = ShufflingErrorReport(epsilon=eps, threshold=threshold, num_sequences=S, per_batch_tv=tvs)
        if eps <= threshold:
            last.threshold_met = True
            return S, last
    last.threshold_met = False
    return S_max, last


def save_schedule(schedule: BatchSchedule, path) -> None:
    with open(path, "w") as f:
        f.write(f"# policy {schedule.policy} batch_size {schedule.batch_size}\n")
        for batch in schedule.batches:
            f.write(" ".join(map(str, np.asarray(batch, dtype=np.int64).tolist())) + "\n")


def load_schedule(path) -> BatchSchedule:
    policy, batch_size, batches = "unknown", 0, []
    with open(path) as f:
        for line in f:
            line = line.strip()
            if not line:
                continue
            if line.startswith("#"):
                parts = line[1:].split()
                if len(parts) >= 4 and parts[0] == "policy":
                    policy, batch_size = parts[1], int(parts[3])
                continue
            batches.append(np.array(line.split(), dtype=np.int64))
    if batch_size == 0 and batches:
        batch_size = max(len(b) for b in batches)
    return BatchSchedule(batches=batches, batch_size=batch_size, policy=policy)
