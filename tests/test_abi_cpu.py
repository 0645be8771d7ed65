"""CPU-side checks: the C-ABI library loads and exports every declared
symbol, and the host logic mirrors the reference (no GPU needed)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT

from oracle import pcg64
from paper_2112_08541_b200 import _lib
from paper_2112_08541_b200.cachesim import CacheConfig, CacheSimReport, amortized_update_ops
from paper_2112_08541_b200.ordering import BatchSchedule, load_schedule, save_schedule
from paper_2112_08541_b200.sampler import AccessTrace, SamplingConfig, load_trace, pcg_states, save_trace

HEADER = os.path.join(ROOT, "include", "bgl_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bgl_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    syms = declared_symbols()
    for s in ("bgl_sample_hop", "bgl_unique_sorted", "bgl_relabel", "bgl_cache_lookup", "bgl_cache_insert",
              "bgl_gather_rows", "bgl_bfs_level", "bgl_interleave", "bgl_pcg64_tables"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = _lib.load(require_cuda=False)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(declared_symbols()) == set(_lib.PROTOTYPES), "ctypes prototypes out of sync with the header"
    assert lib.bgl_abi_version() == 1


def test_library_error_path_without_gpu():
    lib = _lib.load(require_cuda=False)
    # argument validation runs before any CUDA call
    assert lib.bgl_gather_rows(None, None, None, 0, None, None, 3, None, 0, 0, None) == _lib.BGL_EINVAL
    assert b"row_bytes" in lib.bgl_last_error()
    with pytest.raises(ValueError):
        _lib.check(_lib.BGL_EINVAL)


def test_configs_mirror_reference_validation():
    with pytest.raises(ValueError):
        SamplingConfig(fanouts=())
    with pytest.raises(ValueError):
        SamplingConfig(fanouts=(3, 0))
    with pytest.raises(ValueError, match="policy"):
        CacheConfig(device_capacity=1, policy="mru")
    with pytest.raises(ValueError):
        CacheConfig(device_capacity=-1)
    with pytest.raises(ValueError):
        CacheConfig(device_capacity=1, num_devices=0)


def test_pcg_states_match_numpy_streams():
    st = pcg_states(7, [0, 3, 11])
    for row, b in zip(st, (0, 3, 11)):
        s, inc = pcg64.stream_state((7, b))
        assert (int(row[0]) << 64 | int(row[1])) == s
        assert (int(row[2]) << 64 | int(row[3])) == inc


def test_report_from_counters_and_ops():
    cfg = CacheConfig(device_capacity=4, num_devices=2, feature_bytes_per_node=400)
    c = np.array([[3, 1, 1, 0, 1, 1, 0, 0], [2, 0, 0, 1, 1, 2, 1, 0]])
    rep = CacheSimReport.from_counters(cfg, c, [np.array([0, 1, 3], np.uint8), np.array([2, 3], np.uint8)])
    assert rep.hit_ratio == pytest.approx(3 / 5)
    assert rep.peer_bytes == 400 and rep.remote_fetch_bytes == 800
    assert rep.outcomes == [["D", "P", "M"], ["H", "M"]]
    assert amortized_update_ops(rep)["insertions_per_batch"] == 1.5


def test_trace_and_schedule_roundtrip(tmp_path):
    tr = AccessTrace(batches=[np.array([1, 5, 9]), np.array([2])])
    save_trace(tr, tmp_path / "t.txt")
    back = load_trace(tmp_path / "t.txt")
    assert all(np.array_equal(a, b) for a, b in zip(tr.batches, back.batches))
    sc = BatchSchedule(batches=[np.array([3, 1]), np.array([2])], batch_size=2, policy="proximity-S2")
    save_schedule(sc, tmp_path / "s.txt")
    back = load_schedule(tmp_path / "s.txt")
    assert back.policy == "proximity-S2" and back.batch_size == 2
    assert [b.tolist() for b in back.batches] == [[3, 1], [2]]


def test_native_power_law_generator_is_bit_exact(golden):
    """bgl_power_law_generate (host code behind the C ABI, no GPU) emits the
    reference generator's edge list: its CSR, train mask and labels equal
    gnnio.graph.generate_power_law's on every golden case (graph.py:218-297)."""
    from oracle import graph_oracle as go
    from paper_2112_08541_b200.graph import power_law_edges
    npz = golden("graphgen")
    for i, ((n, d, seed, nl), (tf, cf)) in enumerate(zip(npz["specs"], npz["fracs"])):
        n, d, seed, nl = int(n), int(d), int(seed), int(nl)
        edges, train, labels = power_law_edges(n, d, seed, float(tf), nl, float(cf))
        off, col = go.csr_from_edges(edges.astype(np.int64), n)
        assert np.array_equal(off, npz[f"off_{i}"]) and np.array_equal(col, npz[f"col_{i}"]), (n, d, seed)
        assert np.array_equal(train, np.unpackbits(npz[f"train_{i}"])[:n].astype(bool))
        assert np.array_equal(labels, npz[f"labels_{i}"].astype(np.int64))


def test_power_law_generator_argument_errors():
    from paper_2112_08541_b200.graph import power_law_edges
    for args, msg in [((1, 1, 0), "n must be"), ((10, 0, 0), "avg_degree must be >= 1"),
                      ((10, 10, 0), "avg_degree must be < n")]:
        with pytest.raises(ValueError, match=msg):
            power_law_edges(*args)
    with pytest.raises(ValueError, match="train_fraction"):
        power_law_edges(10, 2, 0, train_fraction=0.0)
    with pytest.raises(ValueError, match="num_labels"):
        power_law_edges(10, 2, 0, num_labels=11)


def test_philox_known_answers_and_restatement():
    """The kernel's Philox4x32-10 (host build of the same function) against
    Random123's known-answer vectors, and the oracle restatement against it."""
    from oracle import counter_sampler as cso
    lib = _lib.load(require_cuda=False)
    kat = [([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
           ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
           ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
            [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1])]
    for ctr, key, want in kat:
        c, k, o = np.array(ctr, np.uint32), np.array(key, np.uint32), np.zeros(4, np.uint32)
        lib.bgl_philox4x32(c.ctypes.data, k.ctypes.data, o.ctypes.data)
        assert o.tolist() == want
        assert cso.philox4x32(ctr, key) == want
