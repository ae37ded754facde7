"""ctypes binding of libqdwhg.so (include/qdwhg.h).

The shared library is built in-tree (paper_2104_14186_b200/lib/libqdwhg.so,
``__graft_entry__.build()`` or ``make -C paper_2104_14186_b200/csrc``).  There
is no fallback: if the library is missing, loading fails loudly.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libqdwhg.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "qdwhg.h")

MAX_TRACE = 64
NUM_STAGES = 8

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double
_U64 = ctypes.c_uint64


class Options(ctypes.Structure):
    _fields_ = [("device", _I32), ("reserved0", _I32), ("arena_bytes", _U64), ("flags", _U64)]


class EigInfo(ctypes.Structure):
    _fields_ = [("mu", _D), ("shift", _D), ("tol", _D), ("c_shift", _D),
                ("rank_index", _I64), ("subspace_size", _I64), ("k", _I64), ("k_found", _I64),
                ("iters_qr", _I64), ("iters_chol", _I64), ("borderline", _I64),
                ("no_savings", _I32), ("randomized", _I32), ("n_trace", _I32), ("subspace_path", _I32),
                ("ell_trace", _D * MAX_TRACE), ("seconds", _D), ("flops", _D),
                ("stage_seconds", _D * NUM_STAGES)]


class SvdInfo(ctypes.Structure):
    _fields_ = [("alpha", _D), ("threshold", _D), ("tol", _D), ("cut", _D),
                ("rank_index", _I64), ("subspace_size", _I64), ("k", _I64), ("k_found", _I64),
                ("iters_qr", _I64), ("iters_chol", _I64),
                ("no_savings", _I32), ("randomized", _I32), ("n_trace", _I32), ("reserved", _I32),
                ("ell_trace", _D * MAX_TRACE), ("seconds", _D), ("flops", _D),
                ("stage_seconds", _D * NUM_STAGES)]


class Accuracy(ctypes.Structure):
    _fields_ = [("orth_left", _D), ("orth_right", _D), ("value_err", _D), ("resid_right", _D),
                ("resid_left", _D), ("n", _I64), ("k", _I64), ("has_value_err", _I32),
                ("reserved", _I32)]


class PolarConfigC(ctypes.Structure):
    _fields_ = [("ell0", _D), ("max_iters", _I64), ("conv_eps", _D), ("chol_switch_c", _D),
                ("force_variant", _I32), ("estimate_ell0", _I32)]


class PolarInfo(ctypes.Structure):
    _fields_ = [("alpha", _D), ("iters_qr", _I64), ("iters_chol", _I64), ("converged", _I32),
                ("n_trace", _I32), ("ell_trace", _D * MAX_TRACE), ("seconds", _D), ("flops", _D)]


class KernelStats(ctypes.Structure):
    _fields_ = [("gemm_launches", _U64), ("other_launches", _U64), ("gemm_timed_launches", _U64),
                ("gemm_seconds", _D), ("gemm_flops", _D), ("gemm_busy_seconds", _D),
                ("dag_timed_launches", _U64), ("dag_seconds", _D), ("dag_flops", _D)]


class EigRequest(ctypes.Structure):
    _fields_ = [("which", _I32), ("iters", _I32), ("c", _D), ("k", _I64), ("tol", _D),
                ("randomize", _I32), ("reserved", _I32), ("seed", _U64)]


class SvdRequest(ctypes.Structure):
    _fields_ = [("mode", _I32), ("randomize", _I32), ("value", _D), ("k", _I64), ("tol", _D),
                ("seed", _U64)]


# every exported symbol with its argtypes (the CPU test checks this list against the header)
SIGNATURES = {
    "qdwhg_create": [_P, _P],
    "qdwhg_destroy": [_P],
    "qdwhg_last_error": [_P],
    "qdwhg_get_launch_count": [_P, _P],
    "qdwhg_synchronize": [_P],
    "qdwhg_set_stream": [_P, _P],
    "qdwhg_profile": [_P, _I32],
    "qdwhg_set_deterministic": [_P, _I32],
    "qdwhg_get_kernel_stats": [_P, _P],
    "qdwhg_partial_eig": [_P, _I64, _P, _I64, _I64, _I32, _D, _U64, _P, _P, _I64, _I64, _P],
    "qdwhg_partial_eig_request": [_P, _I64, _P, _I64, _P, _P, _P, _I64, _I64, _P],
    "qdwhg_partial_svd": [_P, _I64, _I64, _P, _I64, _D, _D, _I32, _U64, _P, _P, _I64, _P, _I64,
                          _I64, _P],
    "qdwhg_partial_svd_request": [_P, _I64, _I64, _P, _I64, _P, _P, _P, _I64, _P, _I64, _I64, _P],
    "qdwhg_polar": [_P, _I64, _I64, _P, _I64, _P, _P, _I64, _P, _I64, _P],
    "qdwhg_run_fixed_iterations": [_P, _I64, _I64, _P, _I64, _D, _I64, _I32, _P, _I64, _P],
    "qdwhg_qdwh_chol_step": [_P, _I64, _I64, _P, _I64, _D, _P, _I64],
    "qdwhg_qdwh_qr_step": [_P, _I64, _I64, _P, _I64, _D, _P, _I64],
    "qdwhg_qr_factor": [_P, _I64, _I64, _P, _I64, _P, _I64, _P, _I64],
    "qdwhg_cholesky": [_P, _I64, _P, _I64, _P, _I64],
    "qdwhg_sym_eig_dense": [_P, _I64, _P, _I64, _P, _P, _I64],
    "qdwhg_svd_dense": [_P, _I64, _I64, _P, _I64, _P, _I64, _P, _P, _I64],
    "qdwhg_two_norm_estimate": [_P, _I64, _I64, _P, _I64, _P],
    "qdwhg_eig_full": [_P, _I64, _P, _I64, _I64, _P, _P, _I64, _P],
    "qdwhg_svd_full": [_P, _I64, _I64, _P, _I64, _I64, _P, _I64, _P, _P, _I64],
    "qdwhg_accuracy_report": [_P, _I64, _I64, _P, _I64, _I64, _P, _I64, _P, _P, _I64, _P, _I32, _P],
    "qdwhg_lanczos_min_bound": [_P, _I64, _P, _I64, _I64, _P],
    "qdwhg_gemm": [_P, _I32, _I32, _I64, _I64, _I64, _D, _P, _I64, _P, _I64, _D, _P, _I64],
    "qdwhg_gemm_ex": [_P, _I32, _I32, _I64, _I64, _I64, _D, _P, _I64, _P, _I64, _D, _P, _I64, _I32,
                      _I32, _D],
    "qdwhg_cholesky_inverse": [_P, _I64, _P, _I64, _P, _I64],
    "qdwhg_cholesky_inverse_fast": [_P, _I64, _P, _I64, _P, _I64],
    "qdwhg_subspace_q2": [_P, _I64, _P, _I64, _D, _P, _P, _P, _I64, _I64],
    "qdwhg_gaussian_matrix": [_P, _I64, _I64, _U64, _P, _I64],
    "qdwhg_dist_unique_id": [_P],
    "qdwhg_dist_create_nccl": [_P, _P, _I32, _I32, _I32, _I32, _P],
    "qdwhg_dist_world_create": [_P, _I32],
    "qdwhg_dist_world_destroy": [_P],
    "qdwhg_dist_create_loopback": [_P, _P, _I32, _I32, _I32, _I32, _P],
    "qdwhg_dist_create_callback": [_P, _P, _I32, _I32, _I32, _I32, _P],
    "qdwhg_dist_destroy": [_P],
    "qdwhg_dist_get_stats": [_P, _P, _P],
    "qdwhg_dist_load": [_P, _I64, _I64, _P, _I64],
    "qdwhg_dist_partial_eig_request": [_P, _I64, _P, _I64, _P, _P, _P, _I64, _I64, _P],
    "qdwhg_dist_partial_svd_request": [_P, _I64, _I64, _P, _I64, _P, _P, _P, _I64, _P, _I64, _I64, _P],
    "qdwhg_dist_pgemm": [_P, _I32, _I32, _I64, _I64, _I64, _D, _P, _I64, _P, _I64, _D, _P, _I64, _P, _I64,
                         _I32],
    "qdwhg_dist_cholesky_inverse": [_P, _I64, _P, _I64, _P, _I64],
    "qdwhg_dist_qr": [_P, _I64, _I64, _P, _I64, _I64, _I64, _P, _P, _I64],
    "qdwhg_halley_weights": [_D, _P],
    "qdwhg_iterations_to_converge": [_D, _D, _I64, _P],
    "qdwhg_choose_shift": [_I64, _P],
}

_LIB = None


def load():
    """Load libqdwhg.so (raises OSError if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"libqdwhg.so not built at {LIB_PATH}; run __graft_entry__.build() "
                          "or make -C paper_2104_14186_b200/csrc")
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        lib.qdwhg_last_error.restype = ctypes.c_char_p
        _LIB = lib
    return _LIB
