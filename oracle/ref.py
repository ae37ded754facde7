"""TEST INFRASTRUCTURE ONLY — ctypes access to the reference itself.

oracle/_ref/libqdwhref.so is the UNMODIFIED reference core
(/root/reference/proj/core/src/*.cpp) plus oracle/ref_shim.cpp, built by
oracle/Makefile with the reference's Release flags.  Used to pin the numpy
oracle, to generate tests/golden/ and as bench.py's ``--impl reference`` /
``cpu_baseline`` (kind "reference") arm.  Absent -> ``available()`` is False.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
INFO_LEN = 64

_P = ctypes.c_void_p
_I = ctypes.c_int64
_D = ctypes.c_double
_U = ctypes.c_uint64


def lib_path() -> str:
    return os.path.join(_HERE, "_ref", "libqdwhref.so")


def available() -> bool:
    return os.path.exists(lib_path())


def _lib():
    global _LIB
    if _LIB is None:
        lib = ctypes.CDLL(lib_path())
        sig = {
            "ref_partial_eig": [_I, _P, _I, ctypes.c_int, _D, _U, _P, _P, _I, _P],
            "ref_partial_svd": [_I, _I, _P, _D, _D, ctypes.c_int, _U, _P, _P, _P, _I, _P],
            "ref_polar": [_I, _I, _P, _D, _I, _D, ctypes.c_int, _P, _P, _P],
            "ref_halley_weights": [_D, _P],
            "ref_iterations_to_converge": [_D, _D, _I, _P],
            "ref_gaussian_matrix": [_I, _I, _U, _P],
            "ref_qr_factor": [_I, _I, _P, _P, _P],
            "ref_cholesky": [_I, _P, _P],
            "ref_sym_eig_dense": [_I, _P, _P, _P],
            "ref_svd_dense": [_I, _I, _P, _P, _P, _P],
            "ref_two_norm_estimate": [_I, _I, _P, _P],
            "ref_lanczos_min_bound": [_I, _P, _I, _P],
            "ref_qdwh_chol_step": [_I, _I, _P, _D, _P],
            "ref_qdwh_qr_step": [_I, _I, _P, _D, _P],
            "ref_run_fixed_iterations": [_I, _I, _P, _D, _I, ctypes.c_int, _P, _P],
            "ref_gen_sym_eig_test": [_I, _I, _U, _P, _P],
            "ref_gen_svd_test": [_I, _U, _P, _P],
            "ref_eig_full": [_I, _P, _I, _P, _P, _P],
            "ref_svd_full": [_I, _I, _P, _I, _P, _P, _P],
            "ref_accuracy_report": [_I, _I, _P, _I, _P, _P, _P, _P, ctypes.c_int, _P],
        }
        for name, args in sig.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        lib.ref_last_error.restype = ctypes.c_char_p
        _LIB = lib
    return _LIB


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise RefError(rc, _lib().ref_last_error().decode())


def _f(a):
    return np.asfortranarray(a, dtype=np.float64)


def _ptr(a):
    return a.ctypes.data


def _unpack_info(info):
    nt = int(info[10])
    return dict(mu_or_alpha=float(info[0]), shift_or_threshold=float(info[1]),
                rank_index=int(info[2]), subspace_size=int(info[3]), k=int(info[4]),
                iters_qr=int(info[5]), iters_chol=int(info[6]), borderline=int(info[7]),
                no_savings=bool(info[8]), randomized=bool(info[9]),
                ell_trace=[float(x) for x in info[11:11 + nt]])


def partial_eig(a, iters=3, randomize=False, tol=0.01, seed=0):
    a = _f(a)
    n = a.shape[0]
    lam = np.zeros(n)
    v = np.zeros((n, n), order="F")
    info = np.zeros(INFO_LEN)
    _check(_lib().ref_partial_eig(n, _ptr(a), iters, int(randomize), tol, seed,
                                  _ptr(lam), _ptr(v), n, _ptr(info)))
    d = _unpack_info(info)
    k = d["k"]
    # v was stored densely as n x k (column-major, leading dim n)
    vk = v.reshape(-1, order="F")[: n * k].reshape((n, k), order="F").copy()
    return lam[:k].copy(), vk, d


def partial_svd(a, s, tol=0.01, randomize=False, seed=0):
    a = _f(a)
    m, n = a.shape
    sig = np.zeros(n)
    u = np.zeros(m * n)
    v = np.zeros(n * n)
    info = np.zeros(INFO_LEN)
    _check(_lib().ref_partial_svd(m, n, _ptr(a), s, tol, int(randomize), seed, _ptr(sig),
                                  _ptr(u), _ptr(v), n, _ptr(info)))
    d = _unpack_info(info)
    k = d["k"]
    return (sig[:k].copy(), u[: m * k].reshape((m, k), order="F").copy(),
            v[: n * k].reshape((n, k), order="F").copy(), d)


def polar(a, ell0=1e-15, max_iters=60, chol_switch_c=100.0, variant=0):
    a = _f(a)
    m, n = a.shape
    up = np.zeros((m, n), order="F")
    h = np.zeros((n, n), order="F")
    info = np.zeros(INFO_LEN)
    _check(_lib().ref_polar(m, n, _ptr(a), ell0, max_iters, chol_switch_c, variant, _ptr(up),
                            _ptr(h), _ptr(info)))
    d = _unpack_info(info)
    return up, h, d


def halley_weights(ell):
    out = np.zeros(5)
    _check(_lib().ref_halley_weights(ell, _ptr(out)))
    return out


def iterations_to_converge(ell0, eps, max_iters=60):
    out = ctypes.c_int64(0)
    _check(_lib().ref_iterations_to_converge(ell0, eps, max_iters, ctypes.byref(out)))
    return out.value


def gaussian_matrix(m, n, seed):
    out = np.zeros((m, n), order="F")
    _check(_lib().ref_gaussian_matrix(m, n, seed, _ptr(out)))
    return out


def qr_factor(a):
    a = _f(a)
    m, n = a.shape
    q = np.zeros((m, m), order="F")
    r = np.zeros((m, n), order="F")
    _check(_lib().ref_qr_factor(m, n, _ptr(a), _ptr(q), _ptr(r)))
    return q, r


def cholesky(z):
    z = _f(z)
    n = z.shape[0]
    w = np.zeros((n, n), order="F")
    _check(_lib().ref_cholesky(n, _ptr(z), _ptr(w)))
    return w


def sym_eig_dense(s):
    s = _f(s)
    n = s.shape[0]
    vals = np.zeros(n)
    vecs = np.zeros((n, n), order="F")
    _check(_lib().ref_sym_eig_dense(n, _ptr(s), _ptr(vals), _ptr(vecs)))
    return vals, vecs


def svd_dense(a):
    a = _f(a)
    m, n = a.shape
    k = min(m, n)
    u = np.zeros((m, k), order="F")
    sig = np.zeros(k)
    v = np.zeros((n, k), order="F")
    _check(_lib().ref_svd_dense(m, n, _ptr(a), _ptr(u), _ptr(sig), _ptr(v)))
    return u, sig, v


def two_norm_estimate(a):
    a = _f(a)
    out = ctypes.c_double(0)
    _check(_lib().ref_two_norm_estimate(a.shape[0], a.shape[1], _ptr(a), ctypes.byref(out)))
    return out.value


def lanczos_min_bound(a, steps=30):
    a = _f(a)
    out = ctypes.c_double(0)
    _check(_lib().ref_lanczos_min_bound(a.shape[0], _ptr(a), steps, ctypes.byref(out)))
    return out.value


def qdwh_chol_step(x, ell):
    x = _f(x)
    out = np.zeros_like(x, order="F")
    _check(_lib().ref_qdwh_chol_step(x.shape[0], x.shape[1], _ptr(x), ell, _ptr(out)))
    return out


def qdwh_qr_step(x, ell):
    x = _f(x)
    out = np.zeros_like(x, order="F")
    _check(_lib().ref_qdwh_qr_step(x.shape[0], x.shape[1], _ptr(x), ell, _ptr(out)))
    return out


def run_fixed_iterations(x0, ell0, iters, variant):
    """variant: 'QrFirst' | 'CholeskyOnly'"""
    x0 = _f(x0)
    out = np.zeros_like(x0, order="F")
    info = np.zeros(INFO_LEN)
    _check(_lib().ref_run_fixed_iterations(x0.shape[0], x0.shape[1], _ptr(x0), ell0, iters,
                                           0 if variant == "QrFirst" else 1, _ptr(out),
                                           _ptr(info)))
    nt = int(info[10])
    return out, dict(ell=float(info[0]), iters_qr=int(info[5]), iters_chol=int(info[6]),
                     ell_trace=[float(x) for x in info[11:11 + nt]])


def gen_sym_eig_test(n, k, seed):
    a = np.zeros((n, n), order="F")
    d = np.zeros(n)
    _check(_lib().ref_gen_sym_eig_test(n, k, seed, _ptr(a), _ptr(d)))
    return a, d


def gen_svd_test(n, seed):
    a = np.zeros((n, n), order="F")
    d = np.zeros(n)
    _check(_lib().ref_gen_svd_test(n, seed, _ptr(a), _ptr(d)))
    return a, d


def eig_full(a, base_size=32):
    """fullsolve.hpp:21 -> (ascending lambda, V, depth)."""
    a = _f(a)
    n = a.shape[0]
    lam = np.zeros(n)
    v = np.zeros((n, n), order="F")
    depth = ctypes.c_int64(0)
    _check(_lib().ref_eig_full(n, a.ctypes.data, base_size, lam.ctypes.data, v.ctypes.data,
                               ctypes.byref(depth)))
    return lam, v, depth.value


def svd_full(a, base_size=32):
    """fullsolve.hpp:24 -> (U, sigma descending, V)."""
    a = _f(a)
    m, n = a.shape
    u = np.zeros((m, n), order="F")
    v = np.zeros((n, n), order="F")
    s = np.zeros(n)
    _check(_lib().ref_svd_full(m, n, a.ctypes.data, base_size, u.ctypes.data, s.ctypes.data,
                               v.ctypes.data))
    return u, s, v


def accuracy_report(a, u, sigma, v, delta=None, paper_pairing=False):
    """metrics.hpp:25-28 -> [orth_left, orth_right, value_err (NaN: none), resid_right, resid_left]."""
    a, u, v = _f(a), _f(u), _f(v)
    sg = np.ascontiguousarray(sigma, dtype=np.float64)
    dl = None if delta is None else np.ascontiguousarray(delta, dtype=np.float64)
    out = np.zeros(5)
    _check(_lib().ref_accuracy_report(a.shape[0], a.shape[1], a.ctypes.data, sg.shape[0], u.ctypes.data,
                                      sg.ctypes.data, v.ctypes.data,
                                      dl.ctypes.data if dl is not None else None, int(paper_pairing),
                                      out.ctypes.data))
    return out
