"""GPU parity of the fused, software-pipelined, graph-captured pipeline:
every batch's distinct set, cache outcome codes, counters and gathered rows
vs the CPU oracle."""

import numpy as np
import pytest
import torch

from oracle import cache_oracle as co
from oracle import features_oracle as fo
from oracle import ordering_oracle as oo
from oracle import sampler_oracle as so

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("use_graph", [False, True])
@pytest.mark.parametrize("where", ["host", "hbm"])
def test_pipeline_matches_oracle(use_graph, where):
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
    feats = synthetic_features(n, dim, seed=2, device_resident=(where == "hbm"))
    cap = n // 10
    nb = 12
    distinct = [so.sample_batch(hg.row_offsets, hg.col_indices, ref_batches[i], fan, seed, i)[2]
                for i in range(nb + 2)]
    ref_cnt, ref_codes = co.FifoEngine(cap, 0, 1).run(distinct)
    cum = np.cumsum(ref_cnt, axis=0)

    pipe = MiniBatchPipeline(dg, fan, b, order, seed, CacheConfig(device_capacity=cap, feature_bytes_per_node=400),
                             feats)
    if use_graph:
        pipe.capture()
    for i in range(nb):
        pipe.step()
        torch.cuda.synchronize()
        assert pipe.last_batch() == i
        assert np.array_equal(pipe.distinct().cpu().numpy(), distinct[i]), i
        assert np.array_equal(pipe.rows().cpu().numpy(), fo.synthetic_features(distinct[i], dim, seed=2)), i
        assert np.array_equal(pipe.codes().cpu().numpy(), ref_codes[i]), i
        # lookup + insert of batch i+2 already ran in this step
        assert np.array_equal(pipe.counters.cpu().numpy()[:7], cum[i + 2]), i

    # reset -> the same epoch again from a cold cache, host-fed seeds, results in pinned host memory
    if use_graph:
        pipe.capture(fed=True)
    pipe.reset()

    def feed(i):
        pipe.feed(i, ref_batches[i])

    pipe.prime(fed=True, feed=feed)
    for i in range(4):
        feed(i + pipe.lookahead)
        pipe.step(fed=True)
        torch.cuda.synchronize()
        ids_h, cnt_h = pipe.host_result(pipe.last_slot())
        assert np.array_equal(ids_h.numpy(), distinct[i]), i
        assert np.array_equal(pipe.codes().cpu().numpy(), ref_codes[i])
        assert np.array_equal(pipe.rows().cpu().numpy(), fo.synthetic_features(distinct[i], dim, seed=2)), i
