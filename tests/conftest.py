import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, GOLDEN):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    return load


def golden_graph(npz, name):
    off = npz[f"g_{name}_off"]
    col = npz[f"g_{name}_col"]
    train = npz[f"g_{name}_train"].astype(bool)
    return off, col, train


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
