"""Shuffling error / S selection on the device vs the reference's goldens
(ordering.py:157-231). TV distances are fp64 sums reduced in a different
order than numpy's pairwise sum: tolerance 1e-12 absolute."""

import numpy as np
import pytest

from conftest import golden_graph
from packing import get

TOL = 1e-12


class G:
    def __init__(self, off, col, train, labels):
        self.row_offsets, self.col_indices, self.train_mask, self.labels = off, col, train, labels
        self.num_nodes = len(off) - 1


def _graph(npz, name):
    off, col, train = golden_graph(npz, name)
    return G(off, col, train, npz[f"g_{name}_labels"])


@pytest.mark.gpu
def test_shuffling_error_matches_reference(golden):
    from paper_2112_08541_b200 import ordering
    npz = golden("shuffle")
    names = list(npz["graph_names"])
    tvs = get(npz, "tvs")
    eps = npz["eps"]
    for c, (gi, kind, S, b, seed) in enumerate(npz["meta"]):
        g = _graph(npz, names[gi])
        sched = ordering.proximity_schedule(g, int(S), int(b), seed=int(seed)) if kind == 0 else \
            ordering.random_shuffle_schedule(g, int(b), seed=int(seed))
        rep = ordering.shuffling_error(sched, g.labels)
        assert np.allclose(rep.per_batch_tv, tvs[c], rtol=0, atol=TOL)
        assert abs(rep.epsilon - eps[c]) <= TOL
    nm = len(npz["meta"])
    for j, (gi, b, M, S_max, seed, S_ref, met) in enumerate(npz["select"]):
        g = _graph(npz, names[gi])
        S, rep = ordering.select_num_sequences(g, int(b), int(M), int(S_max), seed=int(seed))
        assert (S, int(rep.threshold_met)) == (S_ref, met)
        assert abs(rep.epsilon - eps[nm + j]) <= TOL


@pytest.mark.gpu
def test_shuffling_error_hand_cases():
    # reference test_ordering.py:170-191: pure batches have TV 0.5; missing label raises
    from paper_2112_08541_b200 import ordering
    sched = ordering.BatchSchedule(batches=[np.array([0, 1]), np.array([2, 3])], batch_size=2, policy="x")
    rep = ordering.shuffling_error(sched, np.array([0, 0, 1, 1]))
    assert np.allclose(rep.per_batch_tv, [0.5, 0.5]) and rep.epsilon == 0.5
    with pytest.raises(ValueError, match="label"):
        ordering.shuffling_error(ordering.BatchSchedule(batches=[np.array([0, 1])], batch_size=1, policy="x"),
                                 np.array([0, -1]))
    assert ordering.shuffling_error_threshold(1000, 4, 1_200_000) == pytest.approx(5.27e-5, rel=1e-2)
