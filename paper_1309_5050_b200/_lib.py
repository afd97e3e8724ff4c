"""ctypes declarations of the C ABI in include/ssa_b200.h (argument marshalling only).

Loading fails loudly when libssa_b200.so is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libssa_b200.so")

SSA_OK = 0
STATUS = {0: "SSA_OK", 1: "SSA_ERR_ARG", 2: "SSA_ERR_WINDOW", 3: "SSA_ERR_EMPTY_KSHAPE", 4: "SSA_ERR_RANK",
          5: "SSA_ERR_NOT_CONVERGED", 6: "SSA_ERR_OOM", 7: "SSA_ERR_CUDA", 8: "SSA_ERR_COMM", 9: "SSA_ERR_STATE"}
SSA_F32, SSA_F64 = 0, 1
PATHS = {"auto": 0, "direct": 1, "fft": 2, "tc": 3}
PATH_NAMES = {v: k for k, v in PATHS.items()}


class ssa_array(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("ld", C.c_int64), ("dtype", C.c_int),
                ("data", C.c_void_p), ("on_device", C.c_int)]


class ssa_window(C.Structure):
    _fields_ = [("lx", C.c_int32), ("ly", C.c_int32), ("wmask", C.c_void_p)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p)


class ssa_comm(C.Structure):
    _fields_ = [("rank", C.c_int), ("world", C.c_int), ("user", C.c_void_p), ("allreduce_sum", ALLREDUCE_FN)]


class ssa_opts(C.Structure):
    _fields_ = [("stream", C.c_void_p), ("path", C.c_int), ("block_k", C.c_int), ("tol", C.c_double),
                ("max_products", C.c_int), ("seed", C.c_uint64), ("comm", C.POINTER(ssa_comm)),
                ("band_y0", C.c_int64), ("band_y1", C.c_int64), ("precision", C.c_int),
                ("ny_global", C.c_int64), ("svd_method", C.c_int)]


class ssa_plan_info_t(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("lx", C.c_int64), ("ly", C.c_int64),
                ("kx", C.c_int64), ("ky", C.c_int64), ("L", C.c_int64), ("K", C.c_int64),
                ("n_valid", C.c_int64), ("n_excluded", C.c_int64), ("path", C.c_int), ("dtype", C.c_int),
                ("full_window", C.c_int), ("full_kshape", C.c_int), ("path_xv", C.c_int), ("path_xtu", C.c_int)]


class ssa_decomp_info(C.Structure):
    _fields_ = [("r_requested", C.c_int32), ("n_converged", C.c_int32), ("block_k", C.c_int32),
                ("n_restarts", C.c_int32), ("n_block_products", C.c_int64), ("n_vector_products", C.c_int64),
                ("max_rel_residual", C.c_double), ("ms_products", C.c_double), ("ms_total", C.c_double),
                ("ms_ritz", C.c_double), ("ms_products_xv", C.c_double), ("ms_products_xtu", C.c_double),
                ("n_products_xv", C.c_int64), ("n_products_xtu", C.c_int64),
                ("n_vectors_xv", C.c_int64), ("n_vectors_xtu", C.c_int64),
                ("sigma_floor_rel", C.c_double), ("n_below_floor", C.c_int32), ("warm_start_cols", C.c_int32),
                ("drop_norm_rel", C.c_double)]


EXPORTS = ["ssa_plan_create", "ssa_plan_destroy", "ssa_plan_info", "ssa_get_weights", "ssa_get_kmask",
           "ssa_matmul", "ssa_decompose", "ssa_get_rank", "ssa_get_sigma", "ssa_get_residuals", "ssa_get_u", "ssa_get_v",
           "ssa_set_triples", "ssa_reconstruct", "ssa_wcor", "ssa_last_error", "ssa_version",
           "ssa_launch_count", "ssa_small_svd", "ssa_bench_tall", "ssa_bench_mma", "ssa_esprit", "ssa_forecast",
           "ssa_release_workspace"]

_lib = None


class SSAError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def load(path: str = SO_PATH):
    """Load the shared library (raises if it is missing: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with `python -m paper_1309_5050_b200.build` "
                          "(the CUDA library is the only implementation; there is no CPU fallback)")
    L = C.CDLL(path)
    p, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
    st = C.c_int
    L.ssa_plan_create.argtypes = [C.POINTER(ssa_array), C.POINTER(ssa_window), p, C.POINTER(ssa_opts), C.POINTER(p)]
    L.ssa_plan_create.restype = st
    L.ssa_plan_destroy.argtypes = [p]; L.ssa_plan_destroy.restype = None
    L.ssa_plan_info.argtypes = [p, C.POINTER(ssa_plan_info_t)]; L.ssa_plan_info.restype = st
    L.ssa_get_weights.argtypes = [p, p, C.c_int]; L.ssa_get_weights.restype = st
    L.ssa_get_kmask.argtypes = [p, p, C.c_int]; L.ssa_get_kmask.restype = st
    L.ssa_matmul.argtypes = [p, C.c_int, p, i64, p, i64, i64, C.c_int]; L.ssa_matmul.restype = st
    L.ssa_decompose.argtypes = [p, i32, C.POINTER(ssa_decomp_info)]; L.ssa_decompose.restype = st
    L.ssa_get_rank.argtypes = [p, C.POINTER(i32)]; L.ssa_get_rank.restype = st
    L.ssa_get_sigma.argtypes = [p, p]; L.ssa_get_sigma.restype = st
    L.ssa_get_residuals.argtypes = [p, p]; L.ssa_get_residuals.restype = st
    L.ssa_get_u.argtypes = [p, p, C.c_int]; L.ssa_get_u.restype = st
    L.ssa_get_v.argtypes = [p, p, C.c_int]; L.ssa_get_v.restype = st
    L.ssa_set_triples.argtypes = [p, i32, p, p, p, C.c_int]; L.ssa_set_triples.restype = st
    L.ssa_reconstruct.argtypes = [p, p, p, i32, C.c_int, p, C.c_int]; L.ssa_reconstruct.restype = st
    L.ssa_wcor.argtypes = [p, p, p, i32, p, p]; L.ssa_wcor.restype = st
    L.ssa_last_error.argtypes = []; L.ssa_last_error.restype = C.c_char_p
    L.ssa_version.argtypes = []; L.ssa_version.restype = C.c_char_p
    L.ssa_launch_count.argtypes = [C.c_int]; L.ssa_launch_count.restype = i64
    L.ssa_release_workspace.argtypes = []; L.ssa_release_workspace.restype = C.c_int
    L.ssa_small_svd.argtypes = [i32, i32, p, C.POINTER(i32), C.POINTER(C.c_double)]
    L.ssa_small_svd.restype = st
    L.ssa_bench_tall.argtypes = [i32, C.c_int64, i32, i32, i32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.ssa_bench_tall.restype = st
    L.ssa_bench_mma.argtypes = [i32, i32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.ssa_bench_mma.restype = st
    L.ssa_esprit.argtypes = [p, p, i32, p, p]; L.ssa_esprit.restype = st
    L.ssa_forecast.argtypes = [p, p, i32, i32, p, i64, C.c_int]; L.ssa_forecast.restype = st
    _lib = L
    return L


def check(status: int, allow=()):
    if status != SSA_OK and status not in allow:
        msg = _lib.ssa_last_error().decode(errors="replace") if _lib else ""
        raise SSAError(status, msg)
    return status
