"""GPU parity of the fused, graph-captured pipeline: every batch's distinct
set, cache outcome counters and gathered rows vs the CPU oracle."""

import numpy as np
import pytest
import torch

from oracle import cache_oracle as co
from oracle import features_oracle as fo
from oracle import ordering_oracle as oo
from oracle import sampler_oracle as so

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("use_graph", [False, True])
def test_pipeline_matches_oracle(use_graph):
    from paper_2112_08541_b200.cachesim import CacheConfig
    from paper_2112_08541_b200.features import synthetic_features
    from paper_2112_08541_b200.graph import generate_power_law_device
    from paper_2112_08541_b200.ordering import proximity_schedule_device
    from paper_2112_08541_b200.pipeline import MiniBatchPipeline

    n, dim, b, fan, seed = 60000, 100, 256, (10, 5), 4
    dg = generate_power_law_device(n, 16, seed=1, train_fraction=0.1, num_labels=8)
    hg = dg.to_host()
    order, _ = proximity_schedule_device(dg, 4, b, seed=seed)
    ref_batches = oo.proximity_schedule(hg.row_offsets, hg.col_indices, hg.train_mask, 4, b, seed)
    assert np.array_equal(order.cpu().numpy(), np.concatenate(ref_batches))
    feats = synthetic_features(n, dim, seed=2)
    cap = n // 10
    pipe = MiniBatchPipeline(dg, fan, b, order, seed, CacheConfig(device_capacity=cap, feature_bytes_per_node=400),
                             feats)
    if use_graph:
        pipe.capture()
    fifo = co.FifoEngine(cap, 0, 1)
    nb = 12
    prev = np.zeros(8, np.int64)
    for i in range(nb):
        pipe.step()
        torch.cuda.synchronize()
        _, _, distinct, _ = so.sample_batch(hg.row_offsets, hg.col_indices, ref_batches[i], fan, seed, i)
        got = pipe.distinct().cpu().numpy()
        assert np.array_equal(got, distinct), i
        rows = pipe.rows().cpu().numpy()
        assert np.array_equal(rows, fo.synthetic_features(distinct, dim, seed=2)), i
        c, codes = fifo.run([distinct], [0])
        assert np.array_equal(pipe.codes().cpu().numpy(), codes[0])
        now = pipe.counters.cpu().numpy()
        assert np.array_equal(now[:7] - prev[:7], c[0]), i
        prev = now
    # reset -> the same epoch again from a cold cache, host-fed seeds
    if use_graph:
        pipe.capture(fed=True)
    pipe.reset()
    fifo = co.FifoEngine(cap, 0, 1)

    def feed(i):
        sb = torch.from_numpy(ref_batches[i].astype(np.int32))
        pipe.fed_seeds[: len(sb)].copy_(sb)
        pipe.fed_count.fill_(len(sb))

    feed(0)
    pipe.prime(fed=True)
    for i in range(4):
        feed(i + 1)
        pipe.step(fed=True)
        torch.cuda.synchronize()
        _, _, distinct, _ = so.sample_batch(hg.row_offsets, hg.col_indices, ref_batches[i], fan, seed, i)
        assert np.array_equal(pipe.distinct().cpu().numpy(), distinct), i
        _, codes = fifo.run([distinct], [0])
        assert np.array_equal(pipe.codes().cpu().numpy(), codes[0])
