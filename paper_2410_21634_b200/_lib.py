"""ctypes binding of libgdiff.so (the C ABI in include/gdiff.h).

The product path has no CPU fallback: if the library or a CUDA device is
missing, every solver raises ``GdiffUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GDIFF_LIB") or os.path.join(HERE, "libgdiff.so")  # override: A/B experiments

GD_OK, GD_ERR_ARG, GD_ERR_CUDA, GD_ERR_OOM, GD_ERR_CAPACITY, GD_ERR_UNSUPPORTED = 0, -1, -2, -3, -4, -5
GD_W_RW, GD_W_CONST, GD_W_ARC = 0, 1, 2
GD_T_DEGREE, GD_T_ARRAY = 0, 1
GD_M_LOCAL_GD, GD_M_LOCAL_SOR, GD_M_LOCAL_CH, GD_M_HK, GD_M_LOCAL_HB = 0, 1, 2, 3, 4
GD_P_PPR, GD_P_KATZ = 0, 1

_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_f64p = C.POINTER(C.c_double)


class GdiffUnavailable(RuntimeError):
    """The CUDA library could not be loaded or no GPU is visible."""


class GdiffError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libgdiff error {code}: {msg}")
        self.code = code


class Operator(C.Structure):
    _fields_ = [("weight_rule", C.c_int32), ("theta_rule", C.c_int32),
                ("beta", C.c_double), ("theta_coeff", C.c_double),
                ("arc_w", _f64p), ("theta", _f64p)]


class Report(C.Structure):
    _fields_ = [("converged", C.c_int32), ("diverged", C.c_int32),
                ("sweeps", C.c_int64), ("total_ops", C.c_int64), ("pushes", C.c_int64),
                ("min_residual", C.c_double), ("support_size", C.c_int64),
                ("n_logs", C.c_int64), ("vol_log", _i64p), ("gamma_log", _f64p),
                ("l1_log", _f64p), ("sign_log", C.POINTER(C.c_int8)),
                ("frontier_sizes", _i64p), ("trace", _i64p), ("trace_len", C.c_int64),
                ("l2_log", _f64p)]


class BatchParams(C.Structure):
    _fields_ = [("method", C.c_int32), ("slots", C.c_int32), ("alpha", C.c_double),
                ("eps", C.c_double), ("max_sweeps", C.c_int64),
                ("frontier_cap", C.c_int64), ("out_cap", C.c_int64),
                ("relabel", C.c_int32), ("problem", C.c_int32), ("omega", C.c_double),
                ("mu", C.c_double), ("L", C.c_double), ("tau", C.c_double),
                ("n_stages", C.c_int64), ("stage_w", _f64p), ("theta_coeff", C.c_double),
                ("want_r", C.c_int32), ("resolve", C.c_int32),
                ("log_sweeps", C.c_int32), ("reserved2", C.c_int32)]


class BatchResult(C.Structure):
    _fields_ = [("sweeps", _i64p), ("total_ops", _i64p), ("pushes", _i64p),
                ("support", _i64p), ("converged", _i32p), ("x_offset", _i64p),
                ("x_count", _i64p), ("x_nodes", _i32p), ("x_vals", _f64p),
                ("x_total", C.c_int64), ("kernel_launches", C.c_int64),
                ("ambiguous", _i32p), ("n_ambiguous", C.c_int64)]


# name -> (restype, argtypes); mirrors include/gdiff.h
SIGNATURES = {
    "gd_last_error": (C.c_char_p, []),
    "gd_version": (C.c_int, []),
    "gd_report_free": (None, [C.POINTER(Report)]),
    "gd_graph_create": (C.c_int, [C.c_int64, _i64p, _i64p, C.c_int64, C.c_int32, C.POINTER(C.c_void_p)]),
    "gd_graph_create_device": (C.c_int, [C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                         C.POINTER(C.c_void_p)]),
    "gd_graph_destroy": (C.c_int, [C.c_void_p]),
    "gd_graph_apply_events": (C.c_int, [C.c_void_p, _i32p, _i64p, _i64p, C.c_int64,
                                        C.POINTER(C.c_void_p)]),
    "gd_graph_apply_events_into": (C.c_int, [C.c_void_p, _i32p, _i64p, _i64p, C.c_int64,
                                             C.c_void_p]),
    "gd_graph_export": (C.c_int, [C.c_void_p, _i64p, _i64p]),
    "gd_graph_info": (C.c_int, [C.c_void_p, _i64p, _i64p, _i64p]),
    "gd_local_gd": (C.c_int, [C.c_void_p, C.POINTER(Operator), _f64p, _f64p, _f64p, C.c_int64,
                              C.c_int32, C.POINTER(Report)]),
    "gd_local_gd_warm": (C.c_int, [C.c_void_p, C.POINTER(Operator), _f64p, _f64p, C.c_int32,
                                   C.c_int64, C.c_int32, C.POINTER(Report)]),
    "gd_local_ch": (C.c_int, [C.c_void_p, C.POINTER(Operator), _f64p, _f64p, _f64p, C.c_double,
                              C.c_double, C.c_int64, C.c_int32, C.POINTER(Report)]),
    "gd_local_hb": (C.c_int, [C.c_void_p, C.POINTER(Operator), _f64p, _f64p, _f64p, C.c_double,
                              C.c_double, C.c_int64, C.c_int32, C.POINTER(Report)]),
    "gd_push_kernel": (C.c_int, [C.c_void_p, C.POINTER(Operator), _f64p, _f64p, _i64p, C.c_int64,
                                 C.c_double, C.c_double, C.c_int32, C.c_int64, C.POINTER(Report)]),
    "gd_hk_push": (C.c_int, [C.c_void_p, C.c_int64, _f64p, C.c_double, _f64p, _f64p, C.c_int64,
                             C.c_int64, C.POINTER(Report)]),
    "gd_gradient_descent": (C.c_int, [C.c_void_p, C.POINTER(Operator), _f64p, _f64p, _f64p,
                                      C.c_int64, C.POINTER(Report)]),
    "gd_spectral_norm": (C.c_int, [C.c_void_p, _f64p, C.c_int64, _f64p]),
    "gd_chebyshev": (C.c_int, [C.c_void_p, C.POINTER(Operator), _f64p, _f64p, _f64p, C.c_double,
                               C.c_double, C.c_int64, C.POINTER(Report)]),
    "gd_hk_taylor": (C.c_int, [C.c_void_p, C.c_int64, _f64p, _f64p, _f64p]),
    "gd_batch_create": (C.c_int, [C.c_void_p, C.POINTER(BatchParams), C.POINTER(C.c_void_p)]),
    "gd_batch_destroy": (C.c_int, [C.c_void_p]),
    "gd_batch_solve_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(BatchResult),
                                        C.c_void_p]),
    "gd_batch_solve_host": (C.c_int, [C.c_void_p, _i64p, C.c_int64, _i64p, _i64p, _i64p, _i32p,
                                      _i64p, _i64p, _i32p, _f64p, C.c_int64, _i64p, C.c_void_p]),
    "gd_batch_fetch_host": (C.c_int, [C.c_void_p, C.c_int64, _i64p, _i64p, _i64p, _i32p, _i64p,
                                      _i64p, _i32p, _f64p, C.c_int64, _i64p, C.c_void_p]),
    "gd_batch_last_kernel_ms": (C.c_int, [C.c_void_p, _f64p]),
    "gd_batch_last_ambiguous": (C.c_int, [C.c_void_p, _i64p]),
    "gd_batch_resolve_stats": (C.c_int, [C.c_void_p, _i64p, _i64p, _f64p]),
    "gd_batch_set_resolve": (C.c_int, [C.c_void_p, C.c_int32]),
    "gd_batch_logs": (C.c_int, [C.c_void_p, C.c_int64, _i64p, _i64p, _f64p]),
    "gd_batch_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), _i64p]),
    "gd_batch_r_device": (C.c_int, [C.c_void_p, C.POINTER(_i64p), C.POINTER(_i64p), C.POINTER(_i32p),
                                    C.POINTER(_f64p), _i64p]),
    "gd_batch_fetch_r_host": (C.c_int, [C.c_void_p, C.c_int64, _i64p, _i64p, _i32p, _f64p, C.c_int64,
                                        _i64p, C.c_void_p]),
    "gd_batch_round_log": (C.c_int, [C.c_void_p, _i64p, C.c_int64, _i64p]),
    "gd_batch_round_phase_log": (C.c_int, [C.c_void_p, _i64p, C.c_int64]),
    "gd_feature_push": (C.c_int, [C.c_void_p, _f64p, _f64p, C.c_double, C.c_double, C.c_int64,
                                  _f64p, C.c_int64, _f64p, _f64p, _i64p, _i64p, _i64p, _i32p]),
    "gd_pairs_create": (C.c_int, [C.c_void_p, C.c_double, C.c_double, _i64p, C.c_int64, C.c_int64,
                                  C.c_int64, C.POINTER(C.c_void_p), _i64p, _i64p, _i64p, _i32p]),
    "gd_pairs_create_ex": (C.c_int, [C.c_void_p, C.c_double, C.c_double, _i64p, C.c_int64,
                                     C.c_int64, C.c_int64, C.c_int32, C.POINTER(C.c_void_p),
                                     _i64p, _i64p, _i64p, _i32p]),
    "gd_pairs_destroy": (C.c_int, [C.c_void_p]),
    "gd_pairs_update": (C.c_int, [C.c_void_p, C.c_void_p, _i32p, _i64p, _i64p, C.c_int64, C.c_int64,
                                  _i64p, _i64p, _i64p, _i32p]),
    "gd_pairs_get": (C.c_int, [C.c_void_p, C.c_int64, _f64p, _f64p]),
    "gd_pairs_device": (C.c_int, [C.c_void_p, C.POINTER(_f64p), C.POINTER(_f64p), _i64p]),
    "gd_pairs_last_kernel_ms": (C.c_int, [C.c_void_p, _f64p]),
    "gd_rmat_keys_device": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                      C.c_double, C.c_double, C.c_double, C.c_void_p, C.c_void_p]),
}

_lock = threading.Lock()
_lib = None


def load(require_gpu: bool = True):
    """Load libgdiff.so; raise GdiffUnavailable when it (or a GPU) is absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise GdiffUnavailable(
                    f"{LIB_PATH} not built; run `python -m paper_2410_21634_b200.build`")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                if os.environ.get("GDIFF_LIB") and not hasattr(lib, name):
                    continue  # (A/B experiments against an older build)
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if require_gpu:
        import torch

        if not torch.cuda.is_available():
            raise GdiffUnavailable("no CUDA device visible; the product path has no CPU fallback")
    return _lib


def check(rc: int) -> None:
    if rc != GD_OK:
        msg = _lib.gd_last_error().decode(errors="replace") if _lib else ""
        raise GdiffError(rc, msg)


def ptr(a: np.ndarray, ct=C.c_double):
    return a.ctypes.data_as(C.POINTER(ct))
