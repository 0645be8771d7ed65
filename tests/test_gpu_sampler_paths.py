"""GPU parity for the sampler's rare paths: hubs mixed into long runs (heavy
gaps), candidate-list overflow and the exact top-k fallback (forced with a
tiny list), the A/B walks (BGL_SAMPLER=slice|hybrid: prep kernel + slice /
lane walk, slice sizes and lane degrees at both extremes; cand|fused) — all bit-exact against the oracle on the same
hub graph."""
import os
import subprocess
import sys

import pytest

import sampler_paths

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def ref_path(tmp_path_factory):
    path = str(tmp_path_factory.mktemp("sampler_paths") / "expected.npz")
    sampler_paths.expected(path)
    return path


def test_hubs_inside_long_runs(ref_path):
    sampler_paths.check(ref_path)


@pytest.mark.parametrize("env", [
    {"BGL_SEG_CAP": "24", "BGL_RUNS_PER_SM": "1"},     # look-back walk: every run 32 parents, lists overflow
    {"BGL_SEG_CAP": "1"},                              # almost every parent takes the fallback
    {"BGL_SEG_OCC": "6x6"},                            # 6 warps x 6 CTAs per SM walk
    {"BGL_SEG_SPLIT": "16", "BGL_RUNS_PER_SM": "1"},   # every 32-parent run hands its second half to idle warps
    {"BGL_SEG_SPLIT": "16", "BGL_SEG_CAP": "24", "BGL_RUNS_PER_SM": "1"},
    {"BGL_SEG_SPLIT": "0"},                            # no split-off
    {"BGL_SAMPLER": "hybrid"},                         # lane walk (deg <= 64) + slices
    {"BGL_SAMPLER": "hybrid", "BGL_LANE_CAP": "12"},   # full lane columns -> exact CTA kernel
    {"BGL_SAMPLER": "hybrid", "BGL_LANE_CAP": "1"},    # almost every lane parent takes the exact kernel
    {"BGL_SAMPLER": "hybrid", "BGL_LANE_DEG": "2048"},  # every light parent walked by one lane
    {"BGL_SAMPLER": "hybrid", "BGL_LANE_DEG": "3", "BGL_SLICE_DRAWS": "256"},
    {"BGL_SAMPLER": "slice"},
    {"BGL_SAMPLER": "slice", "BGL_SEG_CAP": "24"},     # slice walk: lists overflow
    {"BGL_SAMPLER": "slice", "BGL_SEG_CAP": "1"},      # almost every parent takes the fallback
    {"BGL_SAMPLER": "slice", "BGL_SLICE_DRAWS": "256"},      # smallest slices: many empty ones behind long parents
    {"BGL_SAMPLER": "slice", "BGL_SLICE_DRAWS": "1000000"},  # one slice per hop: many 32-parent groups per slice
    {"BGL_SAMPLER": "slice", "BGL_SLICE_DRAWS": "300", "BGL_SEG_CAP": "24"},
    {"BGL_SAMPLER": "cand"},
    {"BGL_SAMPLER": "fused", "BGL_RUNS_PER_SM": "2"},
])
def test_rare_paths_under_env(env, ref_path):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, os.path.join(HERE, "sampler_paths.py"), ref_path], env=e,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-4000:]
