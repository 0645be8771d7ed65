"""bench.py's launch contract on the CPU: the reference arm (`--impl
reference`) runs the reference's CPU path without the product library or
CUDA, under torchrun only rank 0 works and prints, and `--gpus N` is the
N-GPU line's n_gpus. (The GPU arms' N>1 launcher is checked on the GPU in
test_gpu_bench_contract.py.)"""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lines(r):
    assert r.returncode == 0, r.stderr[-4000:]
    return [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_reference_arm_is_isolated_from_the_product():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "4", "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    (d,) = _lines(r)
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["value"] > 0
    assert d["timed_batches"] % d["cpu_baseline"]["cores"] == 0 and d["timed_batches"] >= 4
    iso = d["isolation"]
    assert iso["product_modules"] == [] and not iso["torch_imported"]
    assert not any("paper_2112_08541_b200" in p for p in iso["repo_so_mapped"])
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["csr_entries"] == 2003324 and d["config"]["batches_per_epoch"] == 10


def test_reference_arm_under_torchrun_two_ranks():
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()),
                        os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--config", "c1",
                        "--steps", "2", "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env=env)
    (d,) = _lines(r)                       # rank 0 alone prints
    assert d["n_gpus"] == 2 and d["impl"] == "reference"
    assert d["config"]["cache_rows_per_gpu"] == 5000 and d["config"]["parallelism"].startswith("dp2")


def test_reference_arm_gpus_flag_without_torchrun():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "c1", "--steps", "2", "--warmup", "3"], cwd=ROOT, capture_output=True, text=True,
                       timeout=900)
    (d,) = _lines(r)
    assert d["n_gpus"] == 2
