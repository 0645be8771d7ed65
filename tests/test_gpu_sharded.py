"""GPU parity of the multi-GPU sharded-cache building blocks on one device:
bgl_partition_by_home / bgl_scatter_rows and home-shard engines (D/P codes,
rows) driven through the exchange protocol by hand (the collective protocol
itself is covered by tests/test_distributed_gloo.py)."""

import numpy as np
import pytest
import torch

from oracle import cache_oracle as co
from oracle import features_oracle as fo

pytestmark = pytest.mark.gpu


def test_partition_and_scatter_kernels():
    from paper_2112_08541_b200.distributed import GpuShardOps
    rng = np.random.default_rng(0)
    for H in (1, 2, 3, 8):
        ids = np.unique(rng.integers(0, 100000, size=5000)).astype(np.int32)
        ops = GpuShardOps(H, len(ids), 16)
        part, pos, counts = ops.partition(torch.from_numpy(ids).cuda())
        part, pos, counts = part.cpu().numpy(), pos.cpu().numpy(), counts.cpu().numpy()
        order = np.argsort(ids % H, kind="stable")
        assert np.array_equal(part, ids[order]) and np.array_equal(pos, order)
        assert np.array_equal(counts, np.bincount(ids % H, minlength=H))
        rows = torch.arange(len(ids) * 4, dtype=torch.float32, device="cuda").view(-1, 4)
        out = torch.empty_like(rows)
        ops.scatter(torch.from_numpy(pos).cuda(), rows, out)
        ref = np.empty((len(ids), 4), np.float32)
        ref[pos] = rows.cpu().numpy()
        assert np.array_equal(out.cpu().numpy(), ref)


def test_compact_codes_kernel():
    """bgl_compact_codes (the worker's own miss list): ascending positions with
    code >= min_code, device count, empty / all / none and multi-tile sizes."""
    from paper_2112_08541_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(3)
    for n, cap in ((0, 16), (1, 16), (1000, 1000), (5000, 9000), (300_001, 400_000)):
        for lo in (0, 2, 4):
            codes = rng.integers(0, 4, size=max(cap, 1)).astype(np.uint8)
            d_codes = torch.from_numpy(codes).cuda()
            n_dev = torch.tensor([n], dtype=torch.int64, device="cuda")
            pos = torch.full((max(cap, 1),), -7, dtype=torch.int32, device="cuda")
            cnt = torch.full((1,), -1, dtype=torch.int64, device="cuda")
            ws = torch.empty(int(lib.bgl_compact_codes_workspace(cap)), dtype=torch.uint8, device="cuda")
            _lib.check(lib.bgl_compact_codes(d_codes.data_ptr(), n_dev.data_ptr(), cap, lo, pos.data_ptr(),
                                             cnt.data_ptr(), ws.data_ptr(), _lib.stream_ptr()))
            want = np.flatnonzero(codes[:n] >= lo)
            c = int(cnt.item())
            assert c == want.size, (n, lo)
            assert np.array_equal(pos[:c].cpu().numpy(), want), (n, lo)


@pytest.mark.parametrize("world", [2, 4])
def test_shard_engines_reproduce_reference_d_device_simulation(world):
    from paper_2112_08541_b200.distributed import GpuShardEngine, GpuShardOps
    from paper_2112_08541_b200.features import synthetic_features
    n, dim, cap = 30000, 32, 700
    feats = synthetic_features(n, dim, seed=6)
    ref_table = fo.synthetic_features(np.arange(n), dim, seed=6)
    rng = np.random.default_rng(9)
    batches = [np.unique(rng.integers(0, 4000 + 300 * i, size=3000)).astype(np.int32) for i in range(4 * world)]
    engines = [GpuShardEngine(h, world, cap, feats, max_batch=3000) for h in range(world)]
    ops = GpuShardOps(world, 3000, dim * 4)
    _, ref_codes = co.FifoEngine(cap, 0, world).run(batches)
    for j in range(len(batches) // world):
        buckets = []
        for w in range(world):                      # every worker partitions its batch
            b = torch.from_numpy(batches[j * world + w]).cuda()
            part, pos, counts = ops.partition(b)
            c = counts.cpu().tolist()
            offs = np.concatenate([[0], np.cumsum(c)])
            buckets.append((part.clone(), pos.clone(), offs))
        rows = [torch.empty((len(batches[j * world + w]), dim), device="cuda") for w in range(world)]
        codes = [torch.empty(len(batches[j * world + w]), dtype=torch.uint8, device="cuda") for w in range(world)]
        for h in range(world):                      # every home serves the round in worker order
            for w in range(world):
                part, pos, offs = buckets[w]
                seg = part[offs[h]:offs[h + 1]]
                r = torch.empty((seg.numel(), dim), device="cuda")
                cd = torch.empty(seg.numel(), dtype=torch.uint8, device="cuda")
                engines[h].serve(seg, w, r, cd)
                p = pos[offs[h]:offs[h + 1]].long()
                rows[w][p] = r
                codes[w][p] = cd
        for w in range(world):
            i = j * world + w
            assert np.array_equal(codes[w].cpu().numpy(), ref_codes[i]), i
            assert np.array_equal(rows[w].cpu().numpy(), ref_table[batches[i]]), i
