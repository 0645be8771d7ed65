"""GPU parity: on-device proximity ordering vs the reference's golden vectors."""

import numpy as np
import pytest

from conftest import golden_graph
from packing import get

from oracle import ordering_oracle as oo

pytestmark = pytest.mark.gpu


class G:
    def __init__(self, off, col, train):
        self.row_offsets, self.col_indices, self.train_mask = off, col, train
        self.num_nodes = len(off) - 1


def _graph(npz, names, gi):
    gname = names[gi] if gi < 100 else f"rnd{gi - 100}"
    return G(*golden_graph(npz, gname))


def test_bfs_sequences_match_reference(golden):
    from paper_2112_08541_b200 import ordering
    npz = golden("ordering")
    names = list(npz["graph_names"])
    seqs = get(npz, "seqs")
    s0 = 0
    for gi, S, seed in npz["seq_meta"]:
        g = _graph(npz, names, gi)
        res = ordering.generate_bfs_sequences(g, int(S), seed=int(seed))
        assert len(res) == S
        for a, b in zip(res, seqs[s0:s0 + S]):
            assert np.array_equal(a, b), (gi, S, seed)
        s0 += S


def test_schedules_match_reference(golden):
    from paper_2112_08541_b200 import ordering
    npz = golden("ordering")
    names = list(npz["graph_names"])
    batches = get(npz, "sched_batches")
    b0 = 0
    for gi, S, b, seed, nb, kind in npz["sched_meta"]:
        g = _graph(npz, names, gi)
        if kind == 0:
            sched = ordering.proximity_schedule(g, int(S), int(b), seed=int(seed))
            assert sched.policy == f"proximity-S{S}"
        else:
            sched = ordering.random_shuffle_schedule(g, int(b), seed=int(seed))
        assert len(sched.batches) == nb
        for x, y in zip(sched.batches, batches[b0:b0 + nb]):
            assert np.array_equal(x, y)
        b0 += nb


def test_form_batches_hand_cases():
    from paper_2112_08541_b200 import ordering
    assert [b.tolist() for b in ordering.form_batches([np.arange(7)], 3).batches] == [[0, 1, 2], [3, 4, 5], [6]]
    assert [b.tolist() for b in ordering.form_batches([np.array([1, 2]), np.array([3, 4])], 2).batches] == [[1, 3], [2, 4]]
    assert ordering.form_batches([np.array([1, 2, 5]), np.array([3])], 2).batches[0].tolist() == [1, 3]
    with pytest.raises(ValueError):
        ordering.form_batches([np.array([1])], 0)


def test_large_generated_graph_matches_oracle():
    from paper_2112_08541_b200 import ordering
    from paper_2112_08541_b200.graph import generate_power_law_device
    dg = generate_power_law_device(200000, 20, seed=2, train_fraction=0.05, num_labels=16)
    hg = dg.to_host()
    got = ordering.proximity_schedule(dg, 4, 1024, seed=3)
    ref = oo.proximity_schedule(hg.row_offsets, hg.col_indices, hg.train_mask, 4, 1024, 3)
    assert len(got.batches) == len(ref)
    for a, b in zip(got.batches, ref):
        assert np.array_equal(a, b)
