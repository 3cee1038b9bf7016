"""ctypes binding of libgabp_b200.so (include/gabp_b200.h).

The product path has exactly one implementation: the CUDA library.  If the shared
object is missing or no CUDA device is usable, every entry point raises -- there is no
CPU fallback anywhere in this package.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GABP_LIB") or os.path.join(_PKG, "lib", "libgabp_b200.so")

GABP_OK = 0
GABP_EINVAL = -1
GABP_ECUDA = -2
GABP_ENOMEM = -3
GABP_EZERODIAG = -4
GABP_ESINGULAR = -5
GABP_EDUP = -6

SCHED_IDS = {"parallel": 0, "broadcast": 2}
GATHER_IDS = {"auto": 0, "message": 1, "recompute": 2, "slice": 3, "rows": 4}

# every symbol include/gabp_b200.h declares (checked by tests/test_host.py)
EXPORTED = (
    "gabp_last_error", "gabp_version", "gabp_device_count", "gabp_release_cached",
    "gabp_state_blown", "gabp_state_gather",
    "gabp_graph_create", "gabp_graph_create_device", "gabp_graph_create_device_ex",
    "gabp_graph_create_dense",
    "gabp_graph_destroy", "gabp_graph_info", "gabp_graph_export", "gabp_graph_set_rhs",
    "gabp_graph_stream",
    "gabp_state_create", "gabp_state_clone", "gabp_state_destroy", "gabp_state_reset",
    "gabp_state_read", "gabp_state_write", "gabp_state_counters",
    "gabp_sweep", "gabp_sweep_serial", "gabp_infer_marginals",
    "gabp_solve", "gabp_solve_device", "gabp_solve_system", "gabp_residual_norm_per_eq",
    "gabp_bench_sweeps", "gabp_graph_create_ex", "gabp_nccl_unique_id", "gabp_dist_attach",
    "gabp_dist_solve_local", "gabp_dist_results", "gabp_small_plan",
)


class GraphInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("num_edges", ctypes.c_int64),
                ("num_tiles", ctypes.c_int64), ("max_degree", ctypes.c_int64),
                ("device", ctypes.c_int32), ("is_dense", ctypes.c_int32),
                ("rhs_norm", ctypes.c_double), ("build_ms", ctypes.c_double),
                ("twin_span", ctypes.c_double), ("num_slices", ctypes.c_int64),
                ("num_slots", ctypes.c_int64), ("slice_variant", ctypes.c_int32),
                ("dia_diagonals", ctypes.c_int32)]


class Options(ctypes.Structure):
    _fields_ = [("epsilon", ctypes.c_double), ("max_iter", ctypes.c_int64),
                ("blowup", ctypes.c_double), ("schedule", ctypes.c_int32),
                ("sweeps_per_poll", ctypes.c_int32), ("rel_residual_tol", ctypes.c_double),
                ("means_history", ctypes.POINTER(ctypes.c_double)),
                ("means_history_rows", ctypes.c_int64),
                ("gather_mode", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class Report(ctypes.Structure):
    _fields_ = [("converged", ctypes.c_int32), ("diverged", ctypes.c_int32),
                ("iterations", ctypes.c_int64), ("n_hist", ctypes.c_int64),
                ("sweeps_launched", ctypes.c_int64), ("messages_sent", ctypes.c_int64),
                ("device_ms", ctypes.c_double), ("final_rel_residual", ctypes.c_double),
                ("residual_probes", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("split_sweeps", ctypes.c_int64), ("dist_layout", ctypes.c_int64),
                ("message_bins", ctypes.c_int64)]


class GabpError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"{message} (gabp error {code})")
        self.code = code


_lib = None

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_dp = ctypes.POINTER(ctypes.c_double)
_lp = ctypes.POINTER(ctypes.c_int64)


def load():
    """Load the CUDA library; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"libgabp_b200.so not found at {LIB_PATH}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (make -C "
            "paper_0810_1119_b200/csrc).  There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    sig = {
        "gabp_last_error": (ctypes.c_char_p, []),
        "gabp_version": (ctypes.c_int, []),
        "gabp_device_count": (ctypes.c_int, [ctypes.POINTER(_i32)]),
        "gabp_graph_create": (ctypes.c_int, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _i32,
                                             ctypes.POINTER(_vp)]),
        "gabp_graph_create_device": (ctypes.c_int, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _i32,
                                                    ctypes.POINTER(_vp)]),
        "gabp_graph_create_dense": (ctypes.c_int, [_i64, _vp, _vp, _i32, ctypes.POINTER(_vp)]),
        "gabp_graph_destroy": (None, [_vp]),
        "gabp_graph_info": (ctypes.c_int, [_vp, ctypes.POINTER(GraphInfo)]),
        "gabp_graph_export": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp]),
        "gabp_graph_set_rhs": (ctypes.c_int, [_vp, _vp]),
        "gabp_graph_stream": (_vp, [_vp]),
        "gabp_state_create": (ctypes.c_int, [_vp, ctypes.POINTER(_vp)]),
        "gabp_state_clone": (ctypes.c_int, [_vp, ctypes.POINTER(_vp)]),
        "gabp_state_destroy": (None, [_vp]),
        "gabp_state_reset": (ctypes.c_int, [_vp]),
        "gabp_state_read": (ctypes.c_int, [_vp, _vp, _vp]),
        "gabp_state_write": (ctypes.c_int, [_vp, _vp, _vp]),
        "gabp_state_counters": (ctypes.c_int, [_vp, ctypes.POINTER(_i64),
                                               ctypes.POINTER(_i64)]),
        "gabp_sweep": (ctypes.c_int, [_vp, _vp, _i32, _dp, ctypes.POINTER(_i64),
                                      ctypes.POINTER(_i32)]),
        "gabp_infer_marginals": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
        "gabp_state_blown": (ctypes.c_int, [_vp, ctypes.c_double, ctypes.POINTER(_i32)]),
        "gabp_state_gather": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp]),
        "gabp_solve": (ctypes.c_int, [_vp, ctypes.POINTER(Options), _vp, _vp, _vp, _vp,
                                      ctypes.POINTER(Report)]),
        "gabp_solve_device": (ctypes.c_int, [_vp, ctypes.POINTER(Options), _vp, _vp,
                                             ctypes.POINTER(Report)]),
        "gabp_solve_system": (ctypes.c_int, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _i32,
                                             ctypes.POINTER(Options), _vp, _vp, _vp, _vp,
                                             ctypes.POINTER(Report)]),
        "gabp_residual_norm_per_eq": (ctypes.c_int, [_vp, _vp, _dp]),
        "gabp_sweep_serial": (ctypes.c_int, [_vp, _vp, _vp, _i64, ctypes.c_double, _dp,
                                             ctypes.POINTER(ctypes.c_int32),
                                             ctypes.POINTER(ctypes.c_int64),
                                             ctypes.POINTER(ctypes.c_int32)]),
        "gabp_bench_sweeps": (ctypes.c_int, [_vp, _i32, _i32, _i64, _dp]),
        "gabp_release_cached": (ctypes.c_int, [_i32]),
        "gabp_graph_create_ex": (ctypes.c_int, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _i64,
                                                _i32, ctypes.POINTER(_vp)]),
        "gabp_graph_create_device_ex": (ctypes.c_int, [_i64, _i64, _vp, _vp, _vp, _vp, _vp,
                                                       _i64, _i64, _i32, ctypes.POINTER(_vp)]),
        "gabp_nccl_unique_id": (ctypes.c_int, [_vp]),
        "gabp_dist_attach": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i64, ctypes.c_double, _i32,
                                            _vp, _vp, _vp, _vp, _vp]),
        "gabp_dist_solve_local": (ctypes.c_int, [_i32, _vp, ctypes.POINTER(Options), _dp]),
        "gabp_dist_results": (ctypes.c_int, [_vp, ctypes.POINTER(Options), _vp, _vp, _vp, _vp,
                                             ctypes.POINTER(Report)]),
        "gabp_small_plan": (ctypes.c_int, [_i64, _vp, _vp, ctypes.POINTER(_i64),
                                           ctypes.POINTER(_i64)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().gabp_last_error().decode(errors="replace")


def check(rc: int) -> None:
    if rc != GABP_OK:
        raise GabpError(rc, last_error())


def ptr(a: np.ndarray | None):
    """Host pointer of a C-contiguous numpy array (None -> NULL)."""
    if a is None:
        return None
    if not a.flags.c_contiguous:
        raise ValueError("array must be C-contiguous")
    return ctypes.c_void_p(a.ctypes.data)


def device_count() -> int:
    c = _i32(0)
    rc = load().gabp_device_count(ctypes.byref(c))
    return int(c.value) if rc == GABP_OK else 0


def default_device() -> int:
    env = os.environ.get("LOCAL_RANK")
    return int(env) if env is not None else 0


def release_cached(device: int | None = None) -> None:
    """Give the device memory the library caches for reuse back to the device
    (gabp_release_cached)."""
    check(load().gabp_release_cached(default_device() if device is None else int(device)))
