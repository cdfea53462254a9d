"""ctypes declarations of include/tc.h.  Argument marshalling only: every step of the batch update
runs inside libtc_b200.so on the GPU.  There is no CPU fallback: if the library is missing this
module raises."""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TC_LIB_PATH") or os.path.join(PKG, "libtc_b200.so")  # override: A/B experiments

TC_OK = 0
TC_EINVAL = -1
TC_ENOMEM = -2
TC_ESELFLOOP = -3
TC_EDUP = -4
TC_EOVERFLOW = -5
TC_ECUDA = -6
TC_ENCCL = -7
TC_ESTATE = -8
TC_EPARSE = -9
TC_EIO = -10
TC_EINTERNAL = -11
TC_INGEST_SKIP_LOOPS = 1
TC_NPHASES = 4
PHASES = ("partition", "pairs", "vertices", "update")
TUNE = {"vbucket_arcs": 0, "vbucket_cap": 2, "vbucket_sort_cap": 4, "small_batch": 6, "split_kernels": 8, "small_index": 10, "event_checked": 12, "pair_filter": 14, "small_index_arcs": 16}

EXPORTS = ["tc_create", "tc_create_shard", "tc_create_rank", "tc_create_ex", "tc_nccl_unique_id", "tc_rank_info", "tc_push_batch", "tc_push_batch_after", "tc_test_draws", "tc_test_philox", "tc_estimate", "tc_reset", "tc_destroy", "tc_closed_sum",
           "tc_estimate_mom", "tc_closed_sum_async", "tc_required_estimators", "tc_group_sums", "tc_get_state", "tc_set_state", "tc_set_counters", "tc_counters", "tc_set_async", "tc_set_graphs", "tc_graph_captures", "tc_tune", "tc_set_mode", "tc_get_event_state", "tc_event_counters", "tc_get_steps", "tc_sync",
           "tc_stream", "tc_profile", "tc_profile_read", "tc_profile_kernels", "tc_kernel_name", "tc_stats", "tc_last_launches", "tc_exact_triangles", "tc_parse_edges", "tc_ingest_file", "tc_strerror",
           "tc_last_error"]

_lib = None


class IngestStats(C.Structure):
    """tc_ingest_stats (include/tc.h)."""
    _fields_ = [("edges", C.c_uint64), ("batches", C.c_uint64), ("lines", C.c_uint64), ("error_line", C.c_uint64),
                ("io_s", C.c_double), ("push_s", C.c_double), ("wait_s", C.c_double), ("wall_s", C.c_double)]


class TCConfig(C.Structure):
    """tc_config (include/tc.h)."""
    _fields_ = [("ngpus", C.c_int), ("devices", C.POINTER(C.c_int)), ("strict_errors", C.c_int), ("graphs", C.c_int),
                ("w_max_hint", C.c_uint64)]


class TCError(RuntimeError):
    def __init__(self, code, where=""):
        self.code = code
        super().__init__(f"{where}: {strerror(code)} ({code})" if where else f"{strerror(code)} ({code})")


def load(path: str = LIB_PATH):
    """Load the CUDA library (raises OSError / ImportError when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the product path has no CPU fallback)")
    L = C.CDLL(path)
    u64, u32, vp, i32 = C.c_uint64, C.c_uint32, C.c_void_p, C.c_int
    sig = {
        "tc_create": (vp, [u64, u64]),
        "tc_create_shard": (vp, [u64, u64, u64, u64, i32, u64]),
        "tc_create_rank": (vp, [u64, u64, i32, i32, vp, i32, u64]),
        "tc_create_ex": (vp, [u64, u64, C.POINTER(TCConfig)]),
        "tc_nccl_unique_id": (i32, [vp]),
        "tc_rank_info": (i32, [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(u64), C.POINTER(u64)]),
        "tc_push_batch": (i32, [vp, vp, u64]),
        "tc_push_batch_after": (i32, [vp, vp, u64, vp]),
        "tc_test_draws": (i32, [vp, vp, vp, vp, vp, u64, u64, vp]),
        "tc_test_philox": (i32, [vp, vp, u64, vp]),
        "tc_estimate": (i32, [vp, C.POINTER(C.c_double)]),
        "tc_reset": (i32, [vp]),
        "tc_destroy": (None, [vp]),
        "tc_closed_sum": (i32, [vp, C.POINTER(u64)]),
        "tc_estimate_mom": (i32, [vp, u32, C.POINTER(C.c_double)]),
        "tc_closed_sum_async": (i32, [vp, vp]),
        "tc_required_estimators": (i32, [C.c_double, C.c_double, u64, u64, u64, C.POINTER(u64)]),
        "tc_group_sums": (i32, [vp, u32, vp]),
        "tc_get_state": (i32, [vp, u64, u64, vp, vp, vp, vp, vp, vp]),
        "tc_set_state": (i32, [vp, u64, u64, vp, vp, vp, vp, vp, vp]),
        "tc_set_counters": (i32, [vp, u64, u32]),
        "tc_counters": (i32, [vp, C.POINTER(u64), C.POINTER(u32)]),
        "tc_set_async": (i32, [vp, i32]),
        "tc_set_graphs": (i32, [vp, i32]),
        "tc_graph_captures": (i32, [vp, C.POINTER(u64)]),
        "tc_tune": (i32, [vp, i32, u64]),
        "tc_set_mode": (i32, [vp, i32]),
        "tc_get_event_state": (i32, [vp, u64, u64, vp, vp, vp]),
        "tc_event_counters": (i32, [vp, vp, i32]),
        "tc_get_steps": (i32, [vp, u64, u64, vp, vp, vp, vp, vp, vp]),
        "tc_sync": (i32, [vp]),
        "tc_stream": (vp, [vp]),
        "tc_profile": (i32, [vp, i32]),
        "tc_profile_read": (i32, [vp, vp, vp, i32]),
        "tc_profile_kernels": (i32, [vp, vp, vp, i32]),
        "tc_kernel_name": (C.c_char_p, [i32]),
        "tc_stats": (i32, [vp, vp, i32]),
        "tc_last_launches": (i32, [vp, C.POINTER(u32)]),
        "tc_exact_triangles": (i32, [vp, u64, C.POINTER(u64), C.POINTER(C.c_double)]),
        "tc_parse_edges": (i32, [vp, u64, i32, i32, vp, u64, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64)]),
        "tc_ingest_file": (i32, [vp, C.c_char_p, u64, i32, C.POINTER(IngestStats)]),
        "tc_strerror": (C.c_char_p, [i32]),
        "tc_last_error": (i32, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def strerror(code: int) -> str:
    try:
        return load().tc_strerror(code).decode()
    except Exception:  # library missing: still produce a message
        return f"error {code}"
