"""ctypes binding of the sm_100a C-ABI library (include/bgl_b200.h).

The product path has no CPU fallback: if `_lib/libbgl_b200.so` is missing or
no CUDA device is visible, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# BGL_LIB_PATH: another build of the same ABI (A/B timing of two builds, tools/hop_bench.py)
LIB_PATH = os.environ.get("BGL_LIB_PATH") or os.path.join(_HERE, "_lib", "libbgl_b200.so")

PCG_TABLE_ROWS = 241   # BGL_PCG_TABLE_ROWS (include/bgl_b200.h)
BGL_OK, BGL_EINVAL, BGL_ECUDA, BGL_ENOMEM, BGL_EUNSUPPORTED = 0, 1, 2, 3, 4

c_i32, c_i64, c_u64, c_sz, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t, ctypes.c_void_p
p_i64 = ctypes.POINTER(ctypes.c_int64)   # host int64 arrays (segment tables)

# name -> (restype, argtypes); must list every symbol of include/bgl_b200.h
PROTOTYPES = {
    "bgl_last_error": (ctypes.c_char_p, []),
    "bgl_abi_version": (ctypes.c_int, []),
    "bgl_host_device_pointer": (ctypes.c_int, [c_vp, ctypes.POINTER(c_vp)]),
    "bgl_host_register": (ctypes.c_int, [c_vp, c_sz]),
    "bgl_host_unregister": (ctypes.c_int, [c_vp]),
    "bgl_pcg64_tables": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp]),
    "bgl_pcg64_draws": (ctypes.c_int, [c_vp, c_i64, c_i64, c_vp, c_vp]),
    "bgl_sample_hop_workspace": (c_sz, [c_i64]),
    "bgl_debug_seg_trace": (ctypes.c_int, [c_vp]),
    "bgl_sample_hop": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                       c_i32, c_vp]),
    "bgl_sample_hop_counter_workspace": (c_sz, [c_i64]),
    "bgl_philox4x32": (None, [c_vp, c_vp, c_vp]),
    "bgl_sample_hop_counter": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp,
                                               c_vp, c_vp]),
    "bgl_comm_account": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "bgl_take_i32": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "bgl_unique_workspace": (c_sz, [c_i64]),
    "bgl_unique_workspace_init": (ctypes.c_int, [c_vp, c_i64, c_vp]),
    "bgl_unique_sorted": (ctypes.c_int, [c_vp, c_i32, p_i64, c_vp, p_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "bgl_relabel": (ctypes.c_int, [c_vp, c_i32, p_i64, c_vp, p_i64, c_i64, c_vp, c_vp, c_vp]),
    "bgl_unique_reset": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_i64, c_vp]),
    "bgl_hash_unique_workspace": (c_sz, [c_i64]),
    "bgl_hash_unique": (ctypes.c_int, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "bgl_key_home": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp]),
    "bgl_cache_create": (ctypes.c_int, [c_i64, c_i32, c_i64, c_i64, c_i64, ctypes.POINTER(c_vp)]),
    "bgl_cache_destroy": (ctypes.c_int, [c_vp]),
    "bgl_cache_reserve_nodes": (ctypes.c_int, [c_vp, c_i64, c_vp]),
    "bgl_cache_reset": (ctypes.c_int, [c_vp, c_vp]),
    "bgl_cache_reserve_batch": (ctypes.c_int, [c_vp, c_i64]),
    "bgl_cache_rows": (c_vp, [c_vp]),
    "bgl_cache_set_shard": (ctypes.c_int, [c_vp, c_i32, c_i32]),
    "bgl_cache_set_home_map": (ctypes.c_int, [c_vp, c_vp]),
    "bgl_cache_remap": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp]),
    "bgl_cache_set_policy": (ctypes.c_int, [c_vp, c_i32]),
    "bgl_cache_update_ordered": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "bgl_cache_export_ordered": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "bgl_cache_lookup": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "bgl_cache_lookup_misses": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "bgl_cache_insert": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "bgl_cache_plan_stride": (c_i64, [c_vp, c_i64]),
    "bgl_cache_insert_plan": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "bgl_cache_copy_rows": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "bgl_cache_copy_rows_indexed": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "bgl_cache_export":(ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "bgl_cache_level_stats": (ctypes.c_int, [c_vp, c_vp]),
    "bgl_trace_append": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp]),
    "bgl_degree_histogram": (ctypes.c_int, [c_vp, c_i64, c_i32, c_i64, c_vp, c_vp, c_vp]),
    "bgl_select_flags": (ctypes.c_int, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp]),
    "bgl_compact_workspace": (c_sz, [c_i64]),
    "bgl_compact_flags": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "bgl_cache_warm": (ctypes.c_int, [c_vp, c_vp, p_i64, c_vp, c_i64, c_vp]),
    "bgl_gather_rows":(ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_i32, c_i32, c_vp]),
    "bgl_gather_list": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i32, c_i32, c_vp]),
    "bgl_gather_spans": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_i32, c_vp]),
    "bgl_synthetic_features": (ctypes.c_int, [c_i64, c_i64, c_i32, c_u64, c_vp, c_vp]),
    "bgl_power_law_edge_bound": (c_i64, [c_i64, c_i64, c_i32]),
    "bgl_power_law_generate": (ctypes.c_int, [c_i64, c_i64, c_i32, ctypes.c_double, c_i64, c_vp, c_vp, c_i64, c_vp,
                                              c_vp]),
    "bgl_bfs_workspace": (c_sz, [c_i64]),
    "bgl_bfs_level": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64,
                                     c_vp, c_vp, c_vp, c_vp]),
    "bgl_select_pending": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "bgl_interleave": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i64, c_vp, c_vp]),
    "bgl_shuffling_workspace": (c_sz, [c_i32]),
    "bgl_shuffling_tv": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "bgl_partition_workspace": (c_sz, [c_i64, c_i32]),
    "bgl_partition_by_home": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "bgl_partition_push": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "bgl_scatter_rows": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "bgl_compact_codes_workspace": (c_sz, [c_i64]),
    "bgl_compact_codes": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "bgl_gather_rows_push": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i32,
                                             c_i32, c_vp]),
    "bgl_push_pairs": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "bgl_host_level_codes": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "bgl_host_level_account": (ctypes.c_int, [c_vp, c_vp, c_vp]),
    "bgl_ipc_get_handle": (ctypes.c_int, [c_vp, c_vp, ctypes.POINTER(c_i64)]),
    "bgl_ipc_open_handle": (ctypes.c_int, [c_vp, ctypes.POINTER(c_vp)]),
    "bgl_ipc_close": (ctypes.c_int, [c_vp]),
    "bgl_d2h_result": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "bgl_stage_batch": (ctypes.c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64,
                                        c_i64, c_vp]),
}

_lib = None


class BGLError(RuntimeError):
    pass


def load(require_cuda: bool = True):
    """Load the library (no CUDA needed just to load / list symbols)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise BGLError(f"CUDA extension not built: {LIB_PATH} missing (run __graft_entry__.build())")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_cuda and not torch.cuda.is_available():
        raise BGLError("no CUDA device visible: the B200 path has no CPU fallback")
    return _lib


def check(status: int) -> None:
    if status == BGL_OK:
        return
    msg = load(require_cuda=False).bgl_last_error().decode(errors="replace")
    if status == BGL_EINVAL:
        raise ValueError(msg)
    if status == BGL_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise BGLError(f"bgl status {status}: {msg}")


def call(name: str, *args):
    check(getattr(load(), name)(*args))


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def host_device_pointer(t: torch.Tensor) -> int:
    """Device alias of a pinned host tensor (zero-copy reads from kernels)."""
    out = c_vp()
    check(load().bgl_host_device_pointer(c_vp(t.data_ptr()), ctypes.byref(out)))
    return out.value
