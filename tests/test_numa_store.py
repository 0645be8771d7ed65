"""Host feature-store placement (features.feature_store_plan / mbind) on the
CPU: the plan follows the box's NUMA layout and /dev/shm capacity."""
import mmap

import pytest

from paper_2112_08541_b200 import features as F


def test_plan_single_node_or_policy():
    plan = F.feature_store_plan(1 << 20, 2, 0)
    assert plan["copies"] >= 1 and plan["numa_nodes"] == len(F.numa_nodes())
    if plan["numa_nodes"] == 1:
        assert plan["policy"] == "single"
    else:
        assert plan["policy"] in ("replicate", "interleave")


def test_plan_falls_back_or_raises_when_shm_is_too_small(monkeypatch):
    monkeypatch.setattr(F, "numa_nodes", lambda: [0, 1])
    monkeypatch.setattr(F.os, "statvfs", lambda p: type("S", (), {"f_bavail": 1, "f_frsize": 4096})())
    plan = F.feature_store_plan(1 << 20, 2, 1)     # 1 MB x 2 private copies fit in RAM
    assert plan["policy"] == "private" and plan["copies"] == 2
    with pytest.raises(MemoryError):
        F.feature_store_plan(1 << 60, 2, 1)


def test_plan_replicates_per_node_when_room(monkeypatch):
    monkeypatch.setattr(F, "numa_nodes", lambda: [0, 1])
    monkeypatch.setattr(F.os, "statvfs", lambda p: type("S", (), {"f_bavail": 1 << 30, "f_frsize": 4096})())
    assert F.feature_store_plan(1 << 30, 8, 1)["policy"] == "replicate"
    assert F.feature_store_plan(1 << 30, 8, 1, mode="interleave")["policy"] == "interleave"


def test_mbind_on_an_anonymous_mapping():
    m = mmap.mmap(-1, 1 << 20)
    import ctypes
    addr = ctypes.addressof(ctypes.c_char.from_buffer(m))
    ok = F.mbind(addr, 1 << 20, F.MPOL_INTERLEAVE, F.numa_nodes())
    assert ok in (True, False)            # containers may refuse the syscall; it must not raise
