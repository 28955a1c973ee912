"""ctypes binding of libgdb200.so -- the C ABI declared in include/gd_capi.h.

The library is built in-tree (paper_2507_11094_b200/libgdb200.so) by
__graft_entry__.build().  There is no CPU fallback: importing the package
works without it, but every store/algorithm call raises if it is missing.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import DeviceError, from_status

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgdb200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "gd_capi.h")

_lib = None
_lock = threading.Lock()

vp = C.c_void_p
i64 = C.c_int64
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
u8p = C.POINTER(C.c_uint8)
f64p = C.POINTER(C.c_double)

# (name, restype, argtypes)
SIGNATURES = [
    ("gd_last_error", C.c_char_p, []),
    ("gd_abi_version", C.c_int, []),
    ("gd_kernel_launches", C.c_int64, []),
    ("gd_graph_create", C.c_int, [i64, vp, vp, vp, i64, C.c_int, C.c_int, C.c_int, i64, C.c_int, C.POINTER(vp)]),
    ("gd_graph_destroy", C.c_int, [vp]),
    ("gd_graph_create_dist", C.c_int, [i64, vp, vp, vp, i64, C.c_int, C.c_int, C.c_int, i64, C.c_int, vp,
                                       C.POINTER(vp)]),
    ("gd_graph_owned_range", C.c_int, [vp, i64p, i64p]),
    ("gd_graph_apply_deletes", C.c_int, [vp, vp, vp, i64, i64p, i64p, vp]),
    ("gd_graph_apply_adds", C.c_int, [vp, vp, vp, vp, i64]),
    ("gd_graph_merge", C.c_int, [vp]),
    ("gd_graph_stats", C.c_int, [vp, i64p, i64p, i64p]),
    ("gd_graph_info", C.c_int, [vp, i64p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), i64p]),
    ("gd_graph_segment_slots", C.c_int, [vp, i64, i64p]),
    ("gd_graph_export_segment", C.c_int, [vp, i64, vp, vp, vp]),
    ("gd_graph_reverse_nnz", C.c_int, [vp, i64p]),
    ("gd_graph_export_reverse", C.c_int, [vp, vp, vp, vp]),
    ("gd_graph_export_reverse_slots", C.c_int, [vp, vp, vp, vp, vp, vp]),
    ("gd_graph_propagate_flags", C.c_int, [vp, vp, i64p]),
    ("gd_graph_stream", C.c_int, [vp, C.POINTER(vp)]),
    ("gd_graph_device_bytes", C.c_int, [vp, i64p]),
    ("gd_sssp_create", C.c_int, [vp, i64, C.POINTER(vp)]),
    ("gd_sssp_create_ex", C.c_int, [vp, i64, i64, C.POINTER(vp)]),
    ("gd_sssp_batch", C.c_int, [vp, vp, vp, vp, vp, i64, i64]),
    ("gd_sssp_batch_device", C.c_int, [vp, vp, vp, vp, vp, i64, i64]),
    ("gd_sssp_read", C.c_int, [vp, vp, vp]),
    ("gd_sssp_destroy", C.c_int, [vp]),
    ("gd_pr_create", C.c_int, [vp, C.c_double, C.c_double, i64, C.POINTER(vp)]),
    ("gd_pr_batch", C.c_int, [vp, vp, vp, vp, vp, i64, i64]),
    ("gd_pr_batch_device", C.c_int, [vp, vp, vp, vp, vp, i64, i64]),
    ("gd_pr_read", C.c_int, [vp, vp, vp]),
    ("gd_pr_rank_device", C.c_int, [vp, C.POINTER(vp)]),
    ("gd_pr_read_affected", C.c_int, [vp, vp]),
    ("gd_pr_destroy", C.c_int, [vp]),
    ("gd_tc_create", C.c_int, [vp, C.POINTER(vp)]),
    ("gd_tc_batch", C.c_int, [vp, vp, vp, vp, vp, i64, i64]),
    ("gd_tc_batch_device", C.c_int, [vp, vp, vp, vp, vp, i64, i64]),
    ("gd_tc_read", C.c_int, [vp, i64p]),
    ("gd_tc_destroy", C.c_int, [vp]),
    ("gd_comm_unique_id", C.c_int, [vp]),
    ("gd_comm_create", C.c_int, [C.c_int, C.c_int, vp, C.c_int, C.POINTER(vp)]),
    ("gd_comm_create_local", C.c_int, [C.c_int, C.c_int, i64, C.c_int, C.POINTER(vp)]),
    ("gd_comm_destroy", C.c_int, [vp]),
    ("gd_pr_set_comm", C.c_int, [vp, vp]),
    ("gd_tc_set_comm", C.c_int, [vp, vp]),
    ("gd_phase_times", C.c_int, [vp, f64p]),
    ("gd_iterations", C.c_int, [vp, i64p]),
    ("gd_kernel_time", C.c_int, [vp, C.c_char_p, f64p, i64p, i64p]),
    ("gd_comm_stats", C.c_int, [vp, i64p]),
    ("gd_sssp_read_async", C.c_int, [vp, vp, vp]),
    ("gd_pr_read_async", C.c_int, [vp, vp]),
    ("gd_pr_run_stream", C.c_int, [vp, vp, vp, vp, vp, i64, i64, i64, vp]),
    ("gd_sssp_run_stream", C.c_int, [vp, vp, vp, vp, vp, i64, i64, i64, vp, vp]),
    ("gd_tc_run_stream", C.c_int, [vp, vp, vp, vp, vp, i64, i64, i64, vp]),
    ("gd_pr_run_stream32", C.c_int, [vp, vp, vp, vp, vp, i64, i64, i64, vp]),
    ("gd_sssp_run_stream32", C.c_int, [vp, vp, vp, vp, vp, i64, i64, i64, vp, vp]),
    ("gd_tc_run_stream32", C.c_int, [vp, vp, vp, vp, vp, i64, i64, i64, vp]),
    ("gd_wait", C.c_int, [vp]),
    ("gd_comm_reset_stats", C.c_int, [vp]),
    ("gd_prim_sort", C.c_int, [C.c_int, vp, vp, i64, C.c_int, C.c_int]),
    ("gd_prim_scan_select", C.c_int, [vp, vp, vp, vp, i64, i64p, C.c_int]),
    ("gd_comm_stats_ex", C.c_int, [vp, i64p]),
    ("gd_kernel_time_total", C.c_int, [vp, C.c_char_p, f64p, i64p, i64p]),
    ("gd_set_profiling", C.c_int, [vp, C.c_int]),
]


def lib():
    """Load libgdb200.so (fails loudly when it has not been built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(the B200 path has no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            for name, res, args in SIGNATURES:
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        raise from_status(rc, lib().gd_last_error().decode(errors="replace"))


def ptr(a):
    """ctypes pointer of a numpy array (or None)."""
    if a is None:
        return None
    return C.c_void_p(a.ctypes.data)
