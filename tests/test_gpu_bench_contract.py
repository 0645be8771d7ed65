"""The bench.py JSON contract the driver parses: both arms on the small C1
config (BASELINE.json configs[0]), every required key present and sane."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bgl_arm_line():
    d = _run("--config", "c1", "--steps", "20", "--warmup", "3")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and abs(d["ms_per_step"] - 1e3 / d["value"]) / d["ms_per_step"] < 0.01
    assert "workload" in d["config"]
    roof = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in roof, k
    assert 0 < roof["frac"] <= 1.05 and abs(roof["achieved"] / roof["peak"] - roof["frac"]) < 0.01
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] in ("port", "reference") and cb["sample"]
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= d["steps"]
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_reference_arm_same_config():
    """Both arms describe the same workload with the same config object (the
    driver compares them); the reference arm itself is tested on the CPU
    (tests/test_bench_launcher.py)."""
    g = _run("--config", "c1", "--steps", "4", "--warmup", "3", "--no-cpu-baseline")
    r = _run("--impl", "reference", "--config", "c1", "--steps", "4", "--warmup", "3")
    assert g["config"] == r["config"]
    assert r["isolation"]["product_modules"] == [] and not r["isolation"]["torch_imported"]


def test_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` without torchrun re-launches itself with two ranks
    (shared-GPU mode when the box has one GPU) and prints ONE line whose
    n_gpus is 2, with the per-rank hit rates."""
    import torch
    d = _run("--gpus", "2", "--config", "c1", "--steps", "4", "--warmup", "3")
    assert d["n_gpus"] == 2 and len(d["per_rank"]) == 2 and d["value"] > 0
    assert d["config"]["parallelism"].startswith("dp2")
    assert 0 <= d["peer_hit_pct"] <= d["hit_pct"] <= 100
    if torch.cuda.device_count() < 2:
        assert d["engine"]["shared_gpu"]
    assert "nvlink" in d["roofline"]
