"""TEST INFRASTRUCTURE ONLY — CPU oracle for the QDWHpartial hot path.

A numpy restatement of the reference algorithm (arXiv 2104.14186 artefact,
/root/reference/proj/core), used ONLY by tests/, ``__graft_entry__.smoke()``
and bench.py's ``cpu_baseline`` / ``--impl reference`` legs as the checker.
The product (paper_2104_14186_b200, libqdwhg.so) never imports this module.

Layering:
  * bit-exact scalar/integer layer (Gaussian counter generator, Halley
    weights) -> oracle/qdwh_oracle.c through ctypes (glibc libm, same as the
    reference); pure-Python fallbacks use ``math`` (also glibc) and are
    bit-identical;
  * algorithm layer (Lanczos bound, power-iteration norm, QDWH steps, fixed
    iterations, polar, partial EIG/SVD) restated step by step with the
    reference's control flow, constants, seeds and edge cases;
  * dense kernels: Householder QR, Cholesky, symmetric EIG and SVD are taken
    from LAPACK through numpy.  LAPACK's dgeqrf uses the same reflector
    convention as the reference (R_jj = -sign(x_0)*||x||, Q = H_0 H_1 ...,
    kernels.cpp:59-71), so Q and R agree with the reference to rounding;
    eigh/svd produce the same mathematical objects as the reference's Jacobi
    solvers (kernels.cpp:148-330) up to rounding and eigenvector sign.
    ``householder_qr_loop`` restates kernels.cpp:41-101 literally for the
    small pinning cases.

Pinned against the reference itself (oracle/_ref/libqdwhref.so, built from the
untouched reference sources) by tests/test_oracle_pins.py and against the
committed golden vectors in tests/golden/ (tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np

EPS = float(np.finfo(np.float64).eps)

_HERE = os.path.dirname(os.path.abspath(__file__))
_CLIB = None


def _clib():
    global _CLIB
    if _CLIB is None:
        path = os.path.join(_HERE, "libqdwh_oracle_c.so")
        if not os.path.exists(path):
            return None
        lib = ctypes.CDLL(path)
        lib.qo_gaussian_range.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_void_p]
        lib.qo_uniform_range.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_void_p]
        lib.qo_halley_weights.argtypes = [ctypes.c_double, ctypes.c_void_p]
        lib.qo_halley_weights.restype = ctypes.c_int
        lib.qo_hash64.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        lib.qo_hash64.restype = ctypes.c_uint64
        _CLIB = lib
    return _CLIB


class NotPositiveDefinite(RuntimeError):
    """matrix.hpp:13-16"""


class NotConverged(RuntimeError):
    """matrix.hpp:19-22"""


# ---------------------------------------------------------------- generator
_M64 = (1 << 64) - 1


def hash64(seed: int, counter: int) -> int:
    """splitmix64 finalizer, kernels.cpp:16-21."""
    z = (seed + (counter + 1) * 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def to_unit(h: int) -> float:
    """(0,1] from the top 53 bits, kernels.cpp:24-26."""
    return float((h >> 11) + 1) * 2.0 ** -53


def normal_draw(seed: int, index: int) -> float:
    """Box-Muller on counters 2i, 2i+1, kernels.cpp:28-32."""
    u1 = to_unit(hash64(seed, 2 * index))
    u2 = to_unit(hash64(seed, 2 * index + 1))
    return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


def gaussian_range(seed: int, first: int, count: int) -> np.ndarray:
    lib = _clib()
    out = np.empty(count, dtype=np.float64)
    if lib is not None:
        lib.qo_gaussian_range(seed & _M64, first, count, out.ctypes.data)
    else:
        for i in range(count):
            out[i] = normal_draw(seed, first + i)
    return out


def uniform_range(seed: int, first: int, count: int) -> np.ndarray:
    lib = _clib()
    out = np.empty(count, dtype=np.float64)
    if lib is not None:
        lib.qo_uniform_range(seed & _M64, first, count, out.ctypes.data)
    else:
        for i in range(count):
            out[i] = to_unit(hash64(seed, first + i))
    return out


def gaussian_matrix(m: int, n: int, seed: int) -> np.ndarray:
    """kernels.cpp:441-447 — column-major entry i is draw i.  Returns an
    (m, n) array whose Fortran-order flattening is the draw sequence."""
    if m < 1 or n < 1:
        raise ValueError("gaussian_matrix: dimensions must be >= 1")
    return gaussian_range(seed, 0, m * n).reshape((n, m)).T.copy(order="F")


# ---------------------------------------------------------------- scalars
@dataclass
class WeightStep:
    """polar.hpp:12-18"""
    a: float
    b: float
    c: float
    ell_in: float
    ell_out: float


def halley_weights(ell: float) -> WeightStep:
    """polar.cpp:12-27 (bit-exact: same libm calls in the same order)."""
    if not (ell > 0.0) or ell > 1.0:
        raise ValueError("halley_weights: ell must be in (0, 1]")
    lib = _clib()
    if lib is not None:
        out = np.empty(5, dtype=np.float64)
        lib.qo_halley_weights(float(ell), out.ctypes.data)
        return WeightStep(*[float(v) for v in out])
    l2 = ell * ell
    dd = math.cbrt(4.0 * (1.0 - l2)) * math.pow(ell, -4.0 / 3.0)
    sqd = math.sqrt(1.0 + dd)
    inner = 8.0 - 4.0 * dd + 8.0 * (2.0 - l2) / (l2 * sqd)
    a = sqd + math.sqrt(inner) / 2.0
    b = (a - 1.0) * (a - 1.0) / 4.0
    c = a + b - 1.0
    return WeightStep(a, b, c, ell, ell * (a + b * l2) / (1.0 + c * l2))


def composed_rational(x: float, ell0: float, iters: int) -> float:
    """polar.cpp:29-38"""
    ell, y = ell0, x
    for _ in range(iters):
        w = halley_weights(ell)
        y = y * (w.a + w.b * y * y) / (1.0 + w.c * y * y)
        ell = w.ell_out
    return y


def iterations_to_converge(ell0: float, eps: float, max_iters: int = 60) -> int:
    """polar.cpp:40-51"""
    ell = ell0
    for k in range(max_iters):
        if abs(ell - 1.0) < eps:
            return k
        ell = halley_weights(ell).ell_out
    if abs(ell - 1.0) < eps:
        return max_iters
    raise NotConverged(f"ell recurrence from {ell0} not within {eps} of 1 after {max_iters} steps")


@dataclass
class ShiftPlan:
    """partial.hpp:15-19"""
    s: float = 0.2
    qdwh_iters: int = 3
    kind: str = "ThreeStep"


def choose_shift(qdwh_iters: int) -> ShiftPlan:
    """partial.cpp:26-30"""
    if qdwh_iters == 2:
        return ShiftPlan(0.875, 2, "TwoStep")
    if qdwh_iters == 3:
        return ShiftPlan(0.2, 3, "ThreeStep")
    raise ValueError("choose_shift: unsupported plan, tabulated iteration counts are 2 and 3")


def detect_deficiency_index(r: np.ndarray, tol: float = 0.01):
    """partial.cpp:32-38 — smallest 1-based i with |R_ii| < tol, else None."""
    if r.shape[0] != r.shape[1]:
        raise ValueError("detect_deficiency_index: R must be square")
    d = np.abs(np.diagonal(r))
    hits = np.nonzero(d < tol)[0]
    return int(hits[0]) + 1 if hits.size else None


# ---------------------------------------------------------------- checks
def require_finite(a: np.ndarray, who: str):
    """matrix.cpp:141-145"""
    if a.size == 0:
        raise ValueError(f"{who}: empty matrix")
    if not np.all(np.isfinite(a)):
        raise ValueError(f"{who}: non-finite entry")


def _asym(a: np.ndarray) -> float:
    return float(np.max(np.abs(a - a.T))) if a.size else 0.0


def require_symmetric(a: np.ndarray, who: str):
    """partial.cpp:15-22"""
    if a.shape[0] != a.shape[1]:
        raise ValueError(f"{who}: matrix not square")
    if _asym(a) > 1e3 * a.shape[0] * EPS * max(1.0, np.linalg.norm(a)):
        raise ValueError(f"{who}: input not symmetric within tolerance")


def symmetrize(a: np.ndarray) -> np.ndarray:
    """matrix.cpp:99-105"""
    out = a + a.T
    out *= 0.5
    return out


# ---------------------------------------------------------------- kernels
def householder_qr_loop(a: np.ndarray):
    """Literal restatement of kernels.cpp:41-101 (small sizes only).
    Returns (q_full, r)."""
    m, n = a.shape
    w = np.array(a, dtype=np.float64, copy=True)
    p = min(m - 1 if m >= 1 else 0, n)
    vs, taus = [], []
    for j in range(p):
        v = w[j:, j].copy()
        normx = math.sqrt(float(np.dot(v, v)))
        tau = 0.0
        if normx > 0.0:
            sign = 1.0 if v[0] >= 0.0 else -1.0
            v[0] += sign * normx
            vv = float(np.dot(v, v))
            if vv > 0.0:
                tau = 2.0 / vv
            s = tau * (v @ w[j:, j:])
            w[j:, j:] -= np.outer(v, s)
            w[j, j] = -sign * normx
        vs.append(v)
        taus.append(tau)
    r = np.triu(w)
    q = np.eye(m)
    for jj in range(len(vs) - 1, -1, -1):
        if taus[jj] == 0.0:
            continue
        v = vs[jj]
        s = taus[jj] * (v @ q[jj:, :])
        q[jj:, :] -= np.outer(v, s)
    return q, r


def qr_factor(a: np.ndarray):
    """kernels.cpp:105-112 — full Q (m x m) and R (m x n).  LAPACK Householder
    (same reflector convention as kernels.cpp:59-71)."""
    require_finite(a, "qr_factor")
    q, r = np.linalg.qr(a, mode="complete")
    return q, r


def qr_trailing_q(a: np.ndarray, c0: int):
    """(Q(:, c0:m), |diag R|-ready R) of the Householder QR of square-or-tall a —
    the columns of kernels.cpp:105-112's full Q that partial.cpp:79/146 keep
    (Q2 = Q(:, ind-1:n)), formed by applying the reflectors to the trailing
    identity columns (LAPACK dgeqrf + dormqr, same reflectors and convention as
    np.linalg.qr, so the same Q columns up to rounding) instead of forming all of
    Q.  Returns (r, form) with form(c0) -> Q(:, c0:m)."""
    import scipy.linalg.lapack as L
    require_finite(a, "qr_factor")
    m, n = a.shape
    qr, tau, work, info = L.dgeqrf(np.asfortranarray(a))
    if info != 0:
        raise RuntimeError(f"dgeqrf info={info}")
    r = np.triu(qr[:n, :]) if m >= n else np.triu(qr)

    def form(c0: int) -> np.ndarray:
        e = np.zeros((m, m - c0), order="F")
        e[c0:, :] = np.eye(m - c0)
        lw = L.dormqr("L", "N", qr, tau, e, -1)[1]
        out, _, info2 = L.dormqr("L", "N", qr, tau, e, max(int(lw[0].real), 1), overwrite_c=1)
        if info2 != 0:
            raise RuntimeError(f"dormqr info={info2}")
        return out

    return r, form


def qr_factor_thin(a: np.ndarray, ncols: int):
    """kernels.cpp:114-122"""
    require_finite(a, "qr_factor")
    if ncols > a.shape[0]:
        raise ValueError("qr_factor_thin: ncols > rows")
    q, r = np.linalg.qr(a, mode="complete")
    return q[:, :ncols].copy(), r


def cholesky(z: np.ndarray) -> np.ndarray:
    """kernels.cpp:124-146 — upper W with Z = W^T W."""
    require_finite(z, "cholesky")
    if z.shape[0] != z.shape[1]:
        raise ValueError("cholesky: matrix not square")
    import scipy.linalg.lapack as L
    w, info = L.dpotrf(np.asfortranarray(z), lower=0, clean=1)
    if info != 0:  # pivot <= 0 (kernels.cpp:136-138)
        raise NotPositiveDefinite(f"cholesky: pivot {info} is not positive")
    return w


def sym_eig_dense(s: np.ndarray):
    """kernels.cpp:148-215 — ascending values, orthonormal vectors."""
    require_finite(s, "sym_eig_dense")
    if s.shape[0] != s.shape[1]:
        raise ValueError("sym_eig_dense: matrix not square")
    norm = np.linalg.norm(s)
    if _asym(s) > 1e3 * s.shape[0] * EPS * max(1.0, norm):
        raise ValueError("sym_eig_dense: input not symmetric within tolerance")
    vals, vecs = np.linalg.eigh(symmetrize(s))
    return vals, vecs


def svd_dense(a: np.ndarray):
    """kernels.cpp:217-330 — (U m x min, sigma descending, V n x min)."""
    require_finite(a, "svd_dense")
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    return u, s, vt.T.copy()


def two_norm_estimate(a: np.ndarray) -> float:
    """kernels.cpp:332-360 — power iteration on A^T A from the seeded start,
    stop on relative change < 1e-3, at most 100 steps; returns 1.05*est."""
    require_finite(a, "two_norm_estimate")
    if np.linalg.norm(a) == 0.0:
        raise ValueError("two_norm_estimate: zero matrix")
    n = a.shape[1]
    v = gaussian_matrix(n, 1, 0x6E6F726D32)[:, 0]
    v = v / np.linalg.norm(v)
    est = 0.0
    for it in range(100):
        y = a @ v
        ny = float(np.linalg.norm(y))
        if ny == 0.0:
            v = np.zeros(n)
            v[it % n] = 1.0
            continue
        z = a.T @ y
        nz = float(np.linalg.norm(z))
        prev, est = est, ny
        if nz == 0.0:
            break
        v = z / nz
        if it > 0 and abs(est - prev) < 1e-3 * est:
            break
    return 1.05 * est


def lanczos_min_bound(a: np.ndarray, steps: int = 30) -> float:
    """kernels.cpp:362-439 — Lanczos with two-pass full reorthogonalisation
    from the seeded start; mu = theta_min - beta_last*|s_last|, x1.1 if < 0."""
    require_finite(a, "lanczos_min_bound")
    if a.shape[0] != a.shape[1]:
        raise ValueError("lanczos_min_bound: matrix not square")
    n = a.shape[0]
    fro = float(np.linalg.norm(a))
    if _asym(a) > 1e3 * n * EPS * max(1.0, fro):
        raise ValueError("lanczos_min_bound: input not symmetric within tolerance")
    if steps < 1:
        raise ValueError("lanczos_min_bound: steps must be >= 1")
    m = min(steps, n)
    v0 = gaussian_matrix(n, 1, 0x6C616E637A)[:, 0]
    q = [v0 / math.sqrt(float(np.dot(v0, v0)))]
    alpha, beta = [], []
    beta_last = 0.0
    breakdown_tol = n * EPS * max(1.0, fro)
    for j in range(m):
        w = a @ q[j]
        alpha.append(float(np.dot(q[j], w)))
        for _ in range(2):
            for qk in q:
                w = w - float(np.dot(qk, w)) * qk
        bj = math.sqrt(float(np.dot(w, w)))
        beta_last = bj
        if j + 1 == m or bj <= breakdown_tol:
            if bj <= breakdown_tol:
                beta_last = 0.0
            break
        beta.append(bj)
        q.append(w / bj)
    k = len(alpha)
    t = np.diag(alpha)
    for i in range(k - 1):
        t[i, i + 1] = t[i + 1, i] = beta[i]
    vals, vecs = np.linalg.eigh(t)
    mu = float(vals[0]) - beta_last * abs(float(vecs[k - 1, 0]))
    if mu < 0.0:
        mu *= 1.1
    return mu


# ---------------------------------------------------------------- QDWH steps
def qdwh_qr_step(x: np.ndarray, w: WeightStep) -> np.ndarray:
    """polar.cpp:53-80 — QR of [sqrt(c) X; I], X+ = (b/c)X + ((a-b/c)/sqrt(c)) Q1 Q2^T."""
    require_finite(x, "qdwh_qr_step")
    m, n = x.shape
    sc = math.sqrt(w.c)
    stacked = np.vstack([sc * x, np.eye(n)])
    q, _ = qr_factor_thin(stacked, n)
    q1, q2 = q[:m], q[m:]
    bc = w.b / w.c
    return bc * x + ((w.a - bc) / sc) * (q1 @ q2.T)


def qdwh_chol_step(x: np.ndarray, w: WeightStep) -> np.ndarray:
    """polar.cpp:82-128 — Z = I + c sym(X^T X), W = chol(Z), X+ = (b/c)X + (a-b/c) X W^-1 W^-T."""
    require_finite(x, "qdwh_chol_step")
    import scipy.linalg as sla
    import scipy.linalg.blas as B
    n = x.shape[1]
    # Z = I + c sym(X^T X): the Gram is symmetric by construction (DSYRK's upper
    # triangle, mirrored), so sym() is the identity on it
    z = B.dsyrk(w.c, np.asfortranarray(x), trans=1, lower=0)
    z = np.triu(z) + np.triu(z, 1).T
    z[np.diag_indices(n)] += 1.0
    wu = cholesky(z)
    # Y W = X  ->  Y = X W^-1 ;  G W^T = Y  ->  G = Y W^-T   (right-side DTRSMs)
    y = B.dtrsm(1.0, wu, np.array(x, order="F", copy=True), side=1, lower=0, trans_a=0)
    g = B.dtrsm(1.0, wu, y, side=1, lower=0, trans_a=1, overwrite_b=1)
    bc = w.b / w.c
    return bc * x + (w.a - bc) * g


@dataclass
class FixedIterResult:
    """polar.hpp:64-70"""
    x: np.ndarray
    ell: float
    ell_trace: list
    iters_qr: int = 0
    iters_chol: int = 0


def run_fixed_iterations(x0: np.ndarray, ell0: float, iters: int, variant: str) -> FixedIterResult:
    """polar.cpp:179-215 — variant 'QrFirst' | 'CholeskyOnly'."""
    require_finite(x0, "run_fixed_iterations")
    if not (ell0 > 0.0) or ell0 > 1.0:
        raise ValueError("run_fixed_iterations: ell0 must be in (0, 1]")
    if iters < 1:
        raise ValueError("run_fixed_iterations: iters must be >= 1")
    symmetric = False
    if x0.shape[0] == x0.shape[1]:
        symmetric = _asym(x0) <= 1e3 * x0.shape[0] * EPS * max(1.0, np.linalg.norm(x0))
    res = FixedIterResult(np.array(x0, copy=True), ell0, [ell0])
    for k in range(iters):
        w = halley_weights(res.ell)
        if variant == "QrFirst" and k == 0:
            res.x = qdwh_qr_step(res.x, w)
            res.iters_qr += 1
        else:
            res.x = qdwh_chol_step(res.x, w)
            res.iters_chol += 1
        if symmetric:
            res.x = symmetrize(res.x)
        res.ell = w.ell_out
        res.ell_trace.append(res.ell)
    return res


@dataclass
class PolarResult:
    """polar.hpp:42-50"""
    up: np.ndarray
    h: np.ndarray
    alpha: float
    iters_qr: int
    iters_chol: int
    ell_trace: list
    converged: bool = True


def polar_decompose(a: np.ndarray, ell0: float = 1e-15, max_iters: int = 60,
                    conv_eps: float = EPS, chol_switch_c: float = 100.0,
                    force_variant: str = "Auto") -> PolarResult:
    """polar.cpp:130-177"""
    require_finite(a, "polar_decompose")
    if a.shape[0] < a.shape[1]:
        raise ValueError("polar_decompose: requires rows >= cols")
    if not (ell0 > 0.0) or ell0 > 1.0:
        raise ValueError("polar_decompose: ell0 must be in (0, 1]")
    alpha = two_norm_estimate(a)
    x = a * (1.0 / alpha)
    ell = ell0 / 1.10
    trace = [ell]
    iq = ic = 0
    stop = 5.0 * conv_eps
    while abs(ell - 1.0) >= stop:
        if iq + ic >= max_iters:
            raise NotConverged(f"polar_decompose: no convergence after {max_iters} iterations")
        w = halley_weights(ell)
        use_chol = w.c <= chol_switch_c
        if force_variant == "QrOnly":
            use_chol = False
        if force_variant == "CholeskyOnly":
            use_chol = True
        if use_chol:
            try:
                x = qdwh_chol_step(x, w)
                ic += 1
            except NotPositiveDefinite:
                if force_variant == "CholeskyOnly":
                    raise
                x = qdwh_qr_step(x, w)
                iq += 1
        else:
            x = qdwh_qr_step(x, w)
            iq += 1
        ell = w.ell_out
        trace.append(ell)
    return PolarResult(x, symmetrize(x.T @ a), alpha, iq, ic, trace)


# ---------------------------------------------------------------- drivers
@dataclass
class PartialEigResult:
    """partial.hpp:29-52 (diagnostics flattened)."""
    lambda_minus: np.ndarray
    v: np.ndarray
    subspace_size: int = 0
    mu: float = 0.0
    shift: float = 0.0
    rank_index: int = 0
    ell_trace: list = field(default_factory=list)
    tol: float = 0.01
    iters_qr: int = 0
    iters_chol: int = 0
    borderline: int = 0
    no_savings: bool = False
    randomized: bool = False

    def count(self):
        return len(self.lambda_minus)


def qdwh_partial_eig(a: np.ndarray, plan: ShiftPlan, use_randomization: bool = False,
                     tol: float = 0.01, seed: int = 0) -> PartialEigResult:
    """partial.cpp:40-99 — Alg. 1: negative eigenpairs of symmetric A."""
    require_finite(a, "qdwh_partial_eig")
    require_symmetric(a, "qdwh_partial_eig")
    n = a.shape[0]
    res = PartialEigResult(np.zeros(0), np.zeros((n, 0)), shift=plan.s, tol=tol,
                           randomized=use_randomization)
    res.mu = lanczos_min_bound(a)
    if res.mu >= 0.0:
        return res
    scale = abs(res.mu)
    a_scaled = symmetrize(a) * (1.0 / scale)
    a_tilde = a_scaled * (1.0 - plan.s) - plan.s * np.eye(n)
    it = run_fixed_iterations(a_tilde, plan.s, plan.qdwh_iters, "CholeskyOnly")
    res.ell_trace, res.iters_qr, res.iters_chol = it.ell_trace, it.iters_qr, it.iters_chol
    b = it.x * 0.5 + 0.5 * np.eye(n)
    if use_randomization:
        b = b @ gaussian_matrix(n, n, seed)
    r, form_q = qr_trailing_q(b, 0)
    ind = detect_deficiency_index(r, tol)
    if ind is None:
        return res
    res.rank_index = ind
    ell = n - ind + 1
    res.subspace_size = ell
    res.no_savings = ell > n // 2
    q2 = form_q(ind - 1)[:, :ell]
    reduced = symmetrize(q2.T @ (a_scaled @ q2))
    vals, vecs = sym_eig_dense(reduced)
    max_abs_ritz = float(np.max(np.abs(vals))) if vals.size else 0.0
    floor = -n * EPS * max_abs_ritz
    k = 0
    while k < ell and vals[k] < 0.0:
        k += 1
    if k == 0:
        return res
    res.lambda_minus = scale * vals[:k]
    res.borderline = int(np.sum(vals[:k] >= floor))
    res.v = q2 @ vecs[:, :k]
    return res


@dataclass
class PartialSvdResult:
    """partial.hpp:59-81 (diagnostics flattened)."""
    u1: np.ndarray
    sigma1: np.ndarray
    v1: np.ndarray
    subspace_size: int = 0
    alpha: float = 0.0
    threshold: float = 0.0
    ell_trace: list = field(default_factory=list)
    tol: float = 0.01
    iters_qr: int = 0
    iters_chol: int = 0
    rank_index: int = 0
    no_savings: bool = False
    randomized: bool = False

    def count(self):
        return len(self.sigma1)


def qdwh_partial_svd(a: np.ndarray, s: float, tol: float = 0.01,
                     use_randomization: bool = False, seed: int = 0) -> PartialSvdResult:
    """partial.cpp:101-158 — Alg. 2: singular triplets with sigma > s*alpha."""
    require_finite(a, "qdwh_partial_svd")
    m, n = a.shape
    if m < n:
        raise ValueError("qdwh_partial_svd: requires rows >= cols")
    if not (s > 0.0) or s >= 1.0:
        raise ValueError("qdwh_partial_svd: threshold s must be in (0, 1)")
    res = PartialSvdResult(np.zeros((m, 0)), np.zeros(0), np.zeros((n, 0)), threshold=s,
                           tol=tol, randomized=use_randomization)
    res.alpha = two_norm_estimate(a)
    a_tilde = a * (1.0 / res.alpha)
    iters = iterations_to_converge(s, 5.0 * EPS)
    x = a_tilde
    if iters > 0:
        variant = "QrFirst" if s < 1e-3 else "CholeskyOnly"
        it = run_fixed_iterations(a_tilde, s, iters, variant)
        x = it.x
        res.ell_trace, res.iters_qr, res.iters_chol = it.ell_trace, it.iters_qr, it.iters_chol
    else:
        res.ell_trace = [s]
    mm = np.eye(n) - symmetrize(x.T @ x)
    if use_randomization:
        mm = mm @ gaussian_matrix(n, n, seed)
    r, form_q = qr_trailing_q(mm, 0)
    ind = detect_deficiency_index(r, tol)
    if ind is None:
        return res
    res.rank_index = ind
    ell = n - ind + 1
    res.subspace_size = ell
    res.no_savings = ell > n // 2
    q2 = form_q(ind - 1)[:, :ell]
    u, sig, v = svd_dense(a @ q2)
    cutoff = s * res.alpha
    k = 0
    while k < sig.size and sig[k] > cutoff:
        k += 1
    if k == 0:
        return res
    res.sigma1 = sig[:k].copy()
    res.u1 = u[:, :k].copy()
    res.v1 = q2 @ v[:, :k]
    return res


# ---------------------------------------------------------------- flop model
# ------------------------------------------------------------------ full spectrum + metrics
_SPLIT_SEED = 0x73706C6974  # fullsolve.cpp:14 kSplitSeed


def _eig_recurse(a: np.ndarray, base: int):
    """fullsolve.cpp:22-72"""
    n = a.shape[0]
    if n <= base:
        lam, v = sym_eig_dense(a)
        return lam, v, 0
    sigma = np.trace(a) / n
    shifted = a - sigma * np.eye(n)
    if np.linalg.norm(shifted) <= 10.0 * n * EPS * max(1.0, abs(sigma)):  # fullsolve.cpp:31-38
        return np.full(n, sigma), np.eye(n), 0
    polar = polar_decompose(shifted, ell0=1e-15)  # fullsolve.cpp:40
    c = symmetrize(-0.5 * polar.up + 0.5 * np.eye(n))
    k = int(round(np.trace(c)))
    if k == 0 or k >= n:
        lam, v = sym_eig_dense(a)
        return lam, v, 0
    q, _ = qr_factor(c @ gaussian_matrix(n, n, _SPLIT_SEED))
    v_lo, v_hi = q[:, :k], q[:, k:]
    lo = _eig_recurse(symmetrize(v_lo.T @ (a @ v_lo)), base)
    hi = _eig_recurse(symmetrize(v_hi.T @ (a @ v_hi)), base)
    return (np.concatenate([lo[0], hi[0]]), np.hstack([v_lo @ lo[1], v_hi @ hi[1]]),
            1 + max(lo[2], hi[2]))


def qdwh_eig_full(a: np.ndarray, base_size: int = 32):
    """fullsolve.cpp:76-80 -> (ascending lambda, V, depth)."""
    require_finite(a, "qdwh_eig_full")
    if a.shape[0] != a.shape[1]:
        raise ValueError("qdwh_eig_full: matrix not square")
    return _eig_recurse(symmetrize(a), max(base_size, 2))


def qdwh_svd_full(a: np.ndarray, base_size: int = 32):
    """fullsolve.cpp:82-103 -> (U, sigma descending, V)."""
    require_finite(a, "qdwh_svd_full")
    if a.shape[0] < a.shape[1]:
        raise ValueError("qdwh_svd_full: requires rows >= cols")
    polar = polar_decompose(a)
    lam, w, _ = qdwh_eig_full(polar.h, base_size)
    u_full = polar.up @ w
    return u_full[:, ::-1].copy(), np.maximum(lam[::-1], 0.0), w[:, ::-1].copy()


def accuracy_report(a, u, sigma, v, delta=None, paper_pairing=False):
    """metrics.cpp:58-100 (Eq. 5-7) -> [orth_left, orth_right, value_err (NaN: none),
    resid_right, resid_left]."""
    a, u, v = (np.asarray(x, dtype=np.float64) for x in (a, u, v))
    sigma = np.asarray(sigma, dtype=np.float64)
    k = sigma.shape[0]
    if u.shape[1] != k or v.shape[1] != k:
        raise ValueError("accuracy_report: sigma length must match U and V columns")
    if u.shape[0] != a.shape[0] or v.shape[0] != a.shape[1]:
        raise ValueError("accuracy_report: factor shapes do not conform with A")
    if paper_pairing and a.shape[0] != a.shape[1]:
        raise ValueError("accuracy_report: paper pairing needs a square A")
    nd = max(a.shape[1], 1)

    def gram_defect(x):  # metrics.cpp:10-24
        return np.linalg.norm(np.eye(x.shape[1]) - x.T @ x)

    def max_pair(x, y, op):  # metrics.cpp:26-55
        r = op @ x - y * sigma[None, :]
        return float(np.max(np.linalg.norm(r, axis=0))) if k else 0.0

    out = np.zeros(5)
    out[0], out[1] = gram_defect(u) / nd, gram_defect(v) / nd
    if delta is None:
        out[2] = np.nan
    else:
        delta = np.asarray(delta, dtype=np.float64)
        num, den = np.sum((sigma - delta) ** 2), np.sum(delta ** 2)
        out[2] = np.sqrt(num / den) if den > 0 else np.sqrt(num)
    if paper_pairing:
        out[4], out[3] = max_pair(u, v, a), max_pair(v, u, a)
    else:
        out[3], out[4] = max_pair(v, u, a), max_pair(u, v, a.T)
    return out


def flops_partial_eig(n: int, ell: int, k: int, it_chol: int, randomized: bool) -> float:
    """Algorithmic FP64 count: SYRK n^3 + POTRF n^3/3 + 2 TRSM 2n^3
    per Cholesky step, GEQRF 4/3 n^3, Q2 formation 2n^2 l - 2l^3/3, A Q2 2n^2 l,
    Q2^T A Q2 2n l^2, small EIG 9 l^3, V 2 n l k, randomized Omega 2n^3."""
    n, l = float(n), float(ell)
    f = it_chol * (10.0 / 3.0) * n ** 3 + 4.0 / 3.0 * n ** 3
    f += 2 * n * n * l - 2 * l ** 3 / 3 + 2 * n * n * l + 2 * n * l * l + 9 * l ** 3 + 2 * n * l * k
    if randomized:
        f += 2 * n ** 3
    return f


def flops_partial_svd(m: int, n: int, ell: int, k: int, it_qr: int, it_chol: int,
                      randomized: bool) -> float:
    """SURVEY.md §8(d) SVD count."""
    m, n, l = float(m), float(n), float(ell)
    f = it_qr * (6 * m * n * n + 8.0 / 3.0 * n ** 3) + it_chol * (3 * m * n * n + n ** 3 / 3)
    f += m * n * n + 4.0 / 3.0 * n ** 3 + 2 * n * n * l - 2 * l ** 3 / 3 + 2 * m * n * l
    f += 6 * m * l * l + 20 * l ** 3 + 2 * n * l * k
    if randomized:
        f += 2 * n ** 3
    return f
