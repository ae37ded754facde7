"""Python mirror of the reference's qdwh:: C++ API, backed by libqdwhg.so.

Names, argument meaning, defaults and error behaviour follow
/root/reference/proj/core/include/qdwh/{polar,partial,kernels}.hpp so the
parity tests read like the reference's own tests:

    std::invalid_argument      -> ValueError
    qdwh::NotPositiveDefinite  -> NotPositiveDefinite
    qdwh::NotConverged         -> NotConverged

Matrices are accepted as numpy arrays (host; the call stages them onto the
GPU — the end-to-end path) or torch CUDA tensors (device-resident; no host
copies).  Results come back in the same kind of container.
Everything runs in libqdwhg.so; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib

EPS = float(np.finfo(np.float64).eps)


class NotPositiveDefinite(RuntimeError):
    """qdwh::NotPositiveDefinite (matrix.hpp:13-16)."""


class NotConverged(RuntimeError):
    """qdwh::NotConverged (matrix.hpp:19-22)."""


class CapacityError(RuntimeError):
    """More values found than the caller's k_cap."""


class CudaError(RuntimeError):
    pass


_STATUS = {1: ValueError, 2: NotPositiveDefinite, 3: NotConverged, 4: CapacityError,
           5: CudaError, 6: RuntimeError, 7: RuntimeError}


# ------------------------------------------------------------------ handle
class Handle:
    """One qdwhg handle (device, stream, workspace arena)."""

    def __init__(self, device: int = -1, arena_bytes: int = 0, deterministic: bool = False):
        self.lib = _lib.load()
        self.h = ctypes.c_void_p()
        opts = _lib.Options(device, 0, arena_bytes, 1 if deterministic else 0)
        rc = self.lib.qdwhg_create(ctypes.byref(self.h), ctypes.byref(opts))
        if rc != 0:
            raise _STATUS.get(rc, RuntimeError)(f"qdwhg_create failed ({rc})")

    def check(self, rc: int):
        if rc != 0:
            msg = self.lib.qdwhg_last_error(self.h).decode()
            raise _STATUS.get(rc, RuntimeError)(msg)

    def launches(self) -> int:
        v = ctypes.c_uint64(0)
        self.check(self.lib.qdwhg_get_launch_count(self.h, ctypes.byref(v)))
        return v.value

    def set_stream(self, stream_ptr: int = 0):
        """Run on a caller CUDA stream (e.g. torch.cuda.current_stream().cuda_stream).

        torch reports its legacy default stream as 0; that is passed as
        cudaStreamLegacy (0x1) so the library orders itself after torch's
        work instead of falling back to its own non-blocking stream."""
        self.check(self.lib.qdwhg_set_stream(self.h, ctypes.c_void_p(stream_ptr or 0x1)))

    def own_stream(self):
        """Back to the handle's own (non-blocking) stream."""
        self.check(self.lib.qdwhg_set_stream(self.h, None))

    def set_deterministic(self, enable: bool = True):
        """Bitwise reproducible mode (QDWHG_FLAG_DETERMINISTIC): tall QR panels
        reduce across CTAs in a fixed order instead of with FP64 atomics."""
        self.check(self.lib.qdwhg_set_deterministic(self.h, int(bool(enable))))

    def profile(self, enable: bool = True):
        """Bracket every DMMA GEMM launch with CUDA events (live kernel timing)."""
        self.check(self.lib.qdwhg_profile(self.h, int(bool(enable))))

    def kernel_stats(self) -> dict:
        st = _lib.KernelStats()
        self.check(self.lib.qdwhg_get_kernel_stats(self.h, ctypes.byref(st)))
        return dict(gemm_launches=st.gemm_launches, other_launches=st.other_launches,
                    gemm_timed_launches=st.gemm_timed_launches, gemm_seconds=st.gemm_seconds,
                    gemm_flops=st.gemm_flops, gemm_busy_seconds=st.gemm_busy_seconds,
                    dag_timed_launches=st.dag_timed_launches, dag_seconds=st.dag_seconds,
                    dag_flops=st.dag_flops)

    def close(self):
        if self.h:
            self.lib.qdwhg_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default = threading.local()


def default_handle() -> Handle:
    h = getattr(_default, "h", None)
    if h is None:
        h = Handle()
        _default.h = h
    return h


# ------------------------------------------------------------------ containers
def _is_torch(a) -> bool:
    try:
        import torch
        return isinstance(a, torch.Tensor)
    except ImportError:
        return False


class _Mat:
    """A column-major FP64 operand: pointer + leading dimension, host or device."""

    def __init__(self, a, *, need_rows=None):
        if _is_torch(a):
            import torch
            t = a
            if t.dtype != torch.float64:
                raise ValueError("expected float64")
            if t.dim() == 1:
                t = t.reshape(-1, 1)
            m, n = t.shape
            if not (t.stride(0) == 1 and (n <= 1 or t.stride(1) >= max(m, 1))):
                t = t.t().contiguous().t()  # column-major copy
            # the library runs on its own stream: order it after torch's queued work
            torch.cuda.current_stream(t.device).synchronize()
            self.obj = t
            self.ptr = t.data_ptr()
            self.ld = max(t.stride(1) if n > 1 else m, 1)
            self.shape = (m, n)
            self.device = True
        else:
            arr = np.asarray(a, dtype=np.float64)
            if arr.ndim == 1:
                arr = arr.reshape(-1, 1)
            arr = np.asfortranarray(arr)
            self.obj = arr
            self.ptr = arr.ctypes.data
            self.ld = max(arr.shape[0], 1)
            self.shape = arr.shape
            self.device = False


def _empty_like_kind(ref: _Mat, m: int, n: int):
    if ref.device:
        import torch
        out = torch.zeros((n, m), dtype=torch.float64, device=ref.obj.device).t()
        # the zero fill (and any clone before it) is queued on torch's stream
        torch.cuda.current_stream(out.device).synchronize()
        return out
    return np.zeros((m, n), dtype=np.float64, order="F")


def _ptr_ld(x):
    if _is_torch(x):
        import torch
        # freshly allocated / cloned buffers: order the library after torch's stream
        torch.cuda.current_stream(x.device).synchronize()
        return x.data_ptr(), max(x.stride(1) if x.shape[1] > 1 else x.shape[0], 1)
    return x.ctypes.data, max(x.shape[0], 1)


# ------------------------------------------------------------------ scalars
@dataclass
class WeightStep:
    """polar.hpp:12-18"""
    a: float
    b: float
    c: float
    ell_in: float
    ell_out: float


def halley_weights(ell: float) -> WeightStep:
    """polar.hpp:22 — dynamically weighted Halley coefficients (host scalar)."""
    lib = _lib.load()
    out = (ctypes.c_double * 5)()
    rc = lib.qdwhg_halley_weights(float(ell), out)
    if rc:
        raise _STATUS.get(rc, RuntimeError)("halley_weights: ell must be in (0, 1]")
    return WeightStep(*list(out))


def composed_rational(x: float, ell0: float, iters: int) -> float:
    """polar.cpp:29-38 (scalar oracle of the matrix map)."""
    ell, y = ell0, x
    for _ in range(iters):
        w = halley_weights(ell)
        y = y * (w.a + w.b * y * y) / (1.0 + w.c * y * y)
        ell = w.ell_out
    return y


def iterations_to_converge(ell0: float, eps: float, max_iters: int = 60) -> int:
    """polar.hpp:30"""
    lib = _lib.load()
    out = ctypes.c_int64(0)
    rc = lib.qdwhg_iterations_to_converge(float(ell0), float(eps), int(max_iters),
                                          ctypes.byref(out))
    if rc:
        raise _STATUS.get(rc, RuntimeError)("iterations_to_converge failed")
    return out.value


@dataclass
class ShiftPlan:
    """partial.hpp:15-19"""
    s: float = 0.2
    qdwh_iters: int = 3
    kind: str = "ThreeStep"


def choose_shift(qdwh_iters: int) -> ShiftPlan:
    """partial.hpp:23"""
    lib = _lib.load()
    s = ctypes.c_double(0)
    rc = lib.qdwhg_choose_shift(int(qdwh_iters), ctypes.byref(s))
    if rc:
        raise ValueError("choose_shift: unsupported plan, tabulated iteration counts are 2 and 3")
    return ShiftPlan(s.value, int(qdwh_iters), "TwoStep" if qdwh_iters == 2 else "ThreeStep")


def detect_deficiency_index(r, tol: float = 0.01) -> Optional[int]:
    """partial.cpp:32-38 (host scan of diag(R))."""
    r = np.asarray(r)
    if r.shape[0] != r.shape[1]:
        raise ValueError("detect_deficiency_index: R must be square")
    hits = np.nonzero(np.abs(np.diagonal(r)) < tol)[0]
    return int(hits[0]) + 1 if hits.size else None


# ------------------------------------------------------------------ results
@dataclass
class PartialEigResult:
    """partial.hpp:39-52 (diagnostics flattened)."""
    lambda_minus: np.ndarray
    v: object
    subspace_size: int = 0
    mu: float = 0.0
    shift: float = 0.0
    rank_index: int = 0
    ell_trace: list = field(default_factory=list)
    tol: float = 0.01
    iters_qr: int = 0
    iters_chol: int = 0
    borderline: int = 0
    subspace_path: int = 0  # 0 Householder QR of B, 1 Cholesky-QR extraction
    no_savings: bool = False
    randomized: bool = False
    c_shift: float = 0.0
    k_found: int = 0
    seconds: float = 0.0
    flops: float = 0.0
    stage_seconds: list = field(default_factory=list)

    def count(self) -> int:
        return len(self.lambda_minus)

    def empty(self) -> bool:
        return self.count() == 0


@dataclass
class PartialSvdResult:
    """partial.hpp:69-81 (diagnostics flattened)."""
    u1: object
    sigma1: np.ndarray
    v1: object
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
    k_found: int = 0
    seconds: float = 0.0
    flops: float = 0.0
    stage_seconds: list = field(default_factory=list)

    def count(self) -> int:
        return len(self.sigma1)

    def empty(self) -> bool:
        return self.count() == 0


def _eig_result(info, lam, v, k):
    return PartialEigResult(
        lambda_minus=np.array(lam[:k]), v=v[:, :k], subspace_size=info.subspace_size,
        mu=info.mu, shift=info.shift, rank_index=info.rank_index,
        ell_trace=list(info.ell_trace[:info.n_trace]), tol=info.tol, iters_qr=info.iters_qr,
        iters_chol=info.iters_chol, borderline=info.borderline, subspace_path=info.subspace_path,
        no_savings=bool(info.no_savings),
        randomized=bool(info.randomized), c_shift=info.c_shift, k_found=info.k_found,
        seconds=info.seconds, flops=info.flops, stage_seconds=list(info.stage_seconds))


def _svd_result(info, sig, u, v, k):
    return PartialSvdResult(
        u1=u[:, :k], sigma1=np.array(sig[:k]), v1=v[:, :k], subspace_size=info.subspace_size,
        alpha=info.alpha, threshold=info.threshold, ell_trace=list(info.ell_trace[:info.n_trace]),
        tol=info.tol, iters_qr=info.iters_qr, iters_chol=info.iters_chol,
        rank_index=info.rank_index, no_savings=bool(info.no_savings),
        randomized=bool(info.randomized), k_found=info.k_found, seconds=info.seconds,
        flops=info.flops, stage_seconds=list(info.stage_seconds))


# ------------------------------------------------------------------ drivers
def qdwh_partial_eig(a, plan: ShiftPlan, use_randomization: bool = False, tol: float = 0.01,
                     seed: int = 0, *, k_cap: Optional[int] = None,
                     handle: Optional[Handle] = None) -> PartialEigResult:
    """partial.hpp:55-57 — negative eigenpairs of the symmetric matrix a (Alg. 1)."""
    h = handle or default_handle()
    A = _Mat(a)
    n = A.shape[0]
    if A.shape[1] != n:
        raise ValueError("qdwh_partial_eig: matrix not square")
    kc = n if k_cap is None else k_cap
    lam = np.zeros(max(kc, 1))
    V = _empty_like_kind(A, n, max(kc, 1))
    vp, ldv = _ptr_ld(V)
    info = _lib.EigInfo()
    h.check(h.lib.qdwhg_partial_eig(h.h, n, A.ptr, A.ld, int(plan.qdwh_iters),
                                    int(bool(use_randomization)), float(tol), int(seed) & (2**64 - 1),
                                    lam.ctypes.data, vp, ldv, kc, ctypes.byref(info)))
    return _eig_result(info, lam, V, info.k)


def partial_eig_request(a, which: str = "largest", c: float = 0.0, k: int = 0, iters: int = 3,
                        tol: float = 0.01, use_randomization: bool = False, seed: int = 0, *,
                        k_cap: Optional[int] = None,
                        handle: Optional[Handle] = None) -> PartialEigResult:
    """Spectrum-fraction front end: 'largest' (eigenvalues above c, B = cI - A),
    'smallest' (below c, B = A - cI) or 'negative' (reference semantics);
    keep the k most extreme by count.  lambda_minus holds eigenvalues of A,
    most extreme first."""
    h = handle or default_handle()
    A = _Mat(a)
    n = A.shape[0]
    which_id = {"negative": 0, "largest": 1, "smallest": 2}[which]
    kc = (k if k > 0 else n) if k_cap is None else k_cap
    lam = np.zeros(max(kc, 1))
    V = _empty_like_kind(A, n, max(kc, 1))
    vp, ldv = _ptr_ld(V)
    req = _lib.EigRequest(which_id, iters, float(c), int(k), float(tol), int(bool(use_randomization)),
                          0, int(seed) & (2**64 - 1))
    info = _lib.EigInfo()
    h.check(h.lib.qdwhg_partial_eig_request(h.h, n, A.ptr, A.ld, ctypes.byref(req), lam.ctypes.data,
                                            vp, ldv, kc, ctypes.byref(info)))
    return _eig_result(info, lam, V, info.k)


def qdwh_partial_svd(a, s: float, tol: float = 0.01, use_randomization: bool = False, seed: int = 0,
                     *, k_cap: Optional[int] = None,
                     handle: Optional[Handle] = None) -> PartialSvdResult:
    """partial.hpp:85-86 — singular triplets with sigma > s * alpha (Alg. 2)."""
    h = handle or default_handle()
    A = _Mat(a)
    m, n = A.shape
    kc = n if k_cap is None else k_cap
    sig = np.zeros(max(kc, 1))
    U = _empty_like_kind(A, m, max(kc, 1))
    V = _empty_like_kind(A, n, max(kc, 1))
    up, ldu = _ptr_ld(U)
    vp, ldv = _ptr_ld(V)
    info = _lib.SvdInfo()
    h.check(h.lib.qdwhg_partial_svd(h.h, m, n, A.ptr, A.ld, float(s), float(tol),
                                    int(bool(use_randomization)), int(seed) & (2**64 - 1),
                                    sig.ctypes.data, up, ldu, vp, ldv, kc, ctypes.byref(info)))
    return _svd_result(info, sig, U, V, info.k)


def partial_svd_request(a, cut: Optional[float] = None, s: Optional[float] = None, k: int = 0,
                        tol: float = 0.01, use_randomization: bool = False, seed: int = 0, *,
                        k_cap: Optional[int] = None,
                        handle: Optional[Handle] = None) -> PartialSvdResult:
    """Absolute-cut (sigma > cut) or relative (sigma > s*alpha) front end with top-k by count."""
    h = handle or default_handle()
    A = _Mat(a)
    m, n = A.shape
    if (cut is None) == (s is None):
        raise ValueError("give exactly one of cut / s")
    req = _lib.SvdRequest(1 if cut is not None else 0, int(bool(use_randomization)),
                          float(cut if cut is not None else s), int(k), float(tol),
                          int(seed) & (2**64 - 1))
    kc = (k if k > 0 else n) if k_cap is None else k_cap
    sig = np.zeros(max(kc, 1))
    U = _empty_like_kind(A, m, max(kc, 1))
    V = _empty_like_kind(A, n, max(kc, 1))
    up, ldu = _ptr_ld(U)
    vp, ldv = _ptr_ld(V)
    info = _lib.SvdInfo()
    h.check(h.lib.qdwhg_partial_svd_request(h.h, m, n, A.ptr, A.ld, ctypes.byref(req),
                                            sig.ctypes.data, up, ldu, vp, ldv, kc,
                                            ctypes.byref(info)))
    return _svd_result(info, sig, U, V, info.k)


# ------------------------------------------------------------------ distributed driver
class LoopbackWorld:
    """In-process world for ranks emulated as threads (tests; qdwhg_dist_world_create)."""

    def __init__(self, nranks: int):
        self.lib = _lib.load()
        self.w = ctypes.c_void_p()
        if self.lib.qdwhg_dist_world_create(ctypes.byref(self.w), int(nranks)) != 0:
            raise RuntimeError("qdwhg_dist_world_create failed")

    def close(self):
        if self.w:
            self.lib.qdwhg_dist_world_destroy(self.w)
            self.w = ctypes.c_void_p()


def dist_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0 creates it and shares it, e.g. over torch.distributed)."""
    lib = _lib.load()
    buf = ctypes.create_string_buffer(128)
    rc = lib.qdwhg_dist_unique_id(buf)
    if rc != 0:
        raise _STATUS.get(rc, RuntimeError)("qdwhg_dist_unique_id failed")
    return buf.raw


class Dist:
    """One rank of the distributed QDWHpartial driver (P x Q grid, 2D block-cyclic
    nb x nb tiles; include/qdwhg.h qdwhg_dist_*).  Every rank calls the same
    methods with its own Handle.  Results: values on every rank, vectors on
    rank 0 (None elsewhere)."""

    def __init__(self, handle: Handle, P: int, Q: int, nb: int = 512, rank: int = 0, *,
                 unique_id: Optional[bytes] = None, world: Optional[LoopbackWorld] = None):
        self.h = handle
        self.lib = handle.lib
        self.P, self.Q, self.nb, self.rank = P, Q, nb, rank
        self.d = ctypes.c_void_p()
        if world is not None:
            rc = self.lib.qdwhg_dist_create_loopback(ctypes.byref(self.d), handle.h, P, Q, nb, rank, world.w)
        else:
            if unique_id is None:
                raise ValueError("Dist: unique_id (NCCL) or world (loopback) required")
            self._uid = ctypes.create_string_buffer(bytes(unique_id), 128)
            rc = self.lib.qdwhg_dist_create_nccl(ctypes.byref(self.d), handle.h, P, Q, nb, rank, self._uid)
        handle.check(rc)
        self._kind = None  # (device, torch device) of the loaded matrix

    def close(self):
        if self.d:
            self.lib.qdwhg_dist_destroy(self.d)
            self.d = ctypes.c_void_p()

    def stats(self) -> dict:
        c, g = ctypes.c_uint64(0), ctypes.c_uint64(0)
        self.h.check(self.lib.qdwhg_dist_get_stats(self.d, ctypes.byref(c), ctypes.byref(g)))
        return dict(collectives=c.value, local_gemms=g.value)

    def load(self, a):
        """Keep this rank's tiles of the full matrix a resident (host or device)."""
        A = _Mat(a)
        self._kind = A
        self.h.check(self.lib.qdwhg_dist_load(self.d, A.shape[0], A.shape[1], A.ptr, A.ld))

    def _out(self, ref, m, n):
        return _empty_like_kind(ref, m, n) if self.rank == 0 else None

    def partial_eig_request(self, a=None, which: str = "largest", c: float = 0.0, k: int = 0, iters: int = 3,
                            tol: float = 0.01, use_randomization: bool = False, seed: int = 0, *,
                            n: Optional[int] = None, k_cap: Optional[int] = None) -> "PartialEigResult":
        A = _Mat(a) if a is not None else None
        ref = A if A is not None else self._kind
        if ref is None:
            raise ValueError("no matrix: pass a or load() one")
        nn = ref.shape[0] if n is None else n
        which_id = {"negative": 0, "largest": 1, "smallest": 2}[which]
        kc = (k if k > 0 else nn) if k_cap is None else k_cap
        lam = np.zeros(max(kc, 1))
        V = self._out(ref, nn, max(kc, 1))
        vp, ldv = _ptr_ld(V) if V is not None else (None, 1)
        req = _lib.EigRequest(which_id, iters, float(c), int(k), float(tol), int(bool(use_randomization)),
                              0, int(seed) & (2**64 - 1))
        info = _lib.EigInfo()
        self.h.check(self.lib.qdwhg_dist_partial_eig_request(
            self.d, nn, A.ptr if A is not None else None, A.ld if A is not None else 0, ctypes.byref(req),
            lam.ctypes.data, vp, ldv, kc, ctypes.byref(info)))
        if A is not None:
            self._kind = A
        return _eig_result(info, lam, V if V is not None else np.zeros((0, max(kc, 1))), info.k)

    def partial_svd_request(self, a=None, cut: Optional[float] = None, s: Optional[float] = None, k: int = 0,
                            tol: float = 0.01, use_randomization: bool = False, seed: int = 0, *,
                            shape=None, k_cap: Optional[int] = None) -> "PartialSvdResult":
        A = _Mat(a) if a is not None else None
        ref = A if A is not None else self._kind
        if ref is None:
            raise ValueError("no matrix: pass a or load() one")
        m, n = ref.shape if shape is None else shape
        if (cut is None) == (s is None):
            raise ValueError("give exactly one of cut / s")
        req = _lib.SvdRequest(1 if cut is not None else 0, int(bool(use_randomization)),
                              float(cut if cut is not None else s), int(k), float(tol), int(seed) & (2**64 - 1))
        kc = (k if k > 0 else n) if k_cap is None else k_cap
        sig = np.zeros(max(kc, 1))
        U = self._out(ref, m, max(kc, 1))
        V = self._out(ref, n, max(kc, 1))
        up, ldu = _ptr_ld(U) if U is not None else (None, 1)
        vp, ldv = _ptr_ld(V) if V is not None else (None, 1)
        info = _lib.SvdInfo()
        self.h.check(self.lib.qdwhg_dist_partial_svd_request(
            self.d, m, n, A.ptr if A is not None else None, A.ld if A is not None else 0, ctypes.byref(req),
            sig.ctypes.data, up, ldu, vp, ldv, kc, ctypes.byref(info)))
        if A is not None:
            self._kind = A
        z = np.zeros((0, max(kc, 1)))
        return _svd_result(info, sig, U if U is not None else z, V if V is not None else z, info.k)

    # ---- distributed building blocks on full host operands (result on rank 0)
    def pgemm(self, a, b, c0=None, alpha=1.0, beta=0.0, trans_a=False, trans_b=False, flags=0):
        A, B = np.asfortranarray(a, dtype=np.float64), np.asfortranarray(b, dtype=np.float64)
        m = A.shape[1] if trans_a else A.shape[0]
        k = A.shape[0] if trans_a else A.shape[1]
        n = B.shape[0] if trans_b else B.shape[1]
        C0 = np.asfortranarray(c0 if c0 is not None else np.zeros((m, n)), dtype=np.float64)
        out = np.zeros((m, n), order="F")
        self.h.check(self.lib.qdwhg_dist_pgemm(self.d, int(trans_a), int(trans_b), m, n, k, float(alpha),
                                               A.ctypes.data, A.shape[0], B.ctypes.data, B.shape[0], float(beta),
                                               C0.ctypes.data, m, out.ctypes.data, m, int(flags)))
        return out if self.rank == 0 else None

    def cholesky_inverse(self, z):
        Z = np.asfortranarray(z, dtype=np.float64)
        n = Z.shape[0]
        out = np.zeros((n, n), order="F")
        self.h.check(self.lib.qdwhg_dist_cholesky_inverse(self.d, n, Z.ctypes.data, n, out.ctypes.data, n))
        return out if self.rank == 0 else None

    def qr(self, x, c0, ell):
        X = np.asfortranarray(x, dtype=np.float64)
        m, n = X.shape
        rd = np.zeros(n)
        q2 = np.zeros((m, ell), order="F")
        self.h.check(self.lib.qdwhg_dist_qr(self.d, m, n, X.ctypes.data, m, int(c0), int(ell), rd.ctypes.data,
                                            q2.ctypes.data, m))
        return rd, (q2 if self.rank == 0 else None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class PolarConfig:
    """polar.hpp:34-40"""
    ell0: float = 1e-15
    max_iters: int = 60
    conv_eps: float = EPS
    chol_switch_c: float = 100.0
    force_variant: str = "Auto"  # Auto | QrOnly | CholeskyOnly
    # (no reference counterpart) ignore ell0 and estimate a lower bound of
    # sigma_min(A)/||A||_2 from the R factor of A
    estimate_ell0: bool = False


@dataclass
class PolarResult:
    """polar.hpp:42-50"""
    up: object
    h: object
    alpha: float
    iters_qr: int
    iters_chol: int
    ell_trace: list
    converged: bool
    seconds: float = 0.0
    flops: float = 0.0


def polar_decompose(a, cfg: Optional[PolarConfig] = None, *,
                    handle: Optional[Handle] = None) -> PolarResult:
    """polar.hpp:60"""
    cfg = cfg or PolarConfig()
    h = handle or default_handle()
    A = _Mat(a)
    m, n = A.shape
    Up = _empty_like_kind(A, m, n)
    H = _empty_like_kind(A, n, n)
    upp, ldu = _ptr_ld(Up)
    hp, ldh = _ptr_ld(H)
    c = _lib.PolarConfigC(cfg.ell0, cfg.max_iters, cfg.conv_eps, cfg.chol_switch_c,
                          {"Auto": 0, "QrOnly": 1, "CholeskyOnly": 2}[cfg.force_variant],
                          int(bool(cfg.estimate_ell0)))
    info = _lib.PolarInfo()
    h.check(h.lib.qdwhg_polar(h.h, m, n, A.ptr, A.ld, ctypes.byref(c), upp, ldu, hp, ldh,
                              ctypes.byref(info)))
    return PolarResult(Up, H, info.alpha, info.iters_qr, info.iters_chol,
                       list(info.ell_trace[:info.n_trace]), bool(info.converged), info.seconds,
                       info.flops)


@dataclass
class FixedIterResult:
    """polar.hpp:64-70"""
    x: object
    ell: float
    ell_trace: list
    iters_qr: int
    iters_chol: int


def run_fixed_iterations(x0, ell0: float, iters: int, variant: str = "CholeskyOnly", *,
                         handle: Optional[Handle] = None) -> FixedIterResult:
    """polar.hpp:74-75 — variant 'QrFirst' | 'CholeskyOnly'."""
    h = handle or default_handle()
    X = _Mat(x0)
    m, n = X.shape
    out = _empty_like_kind(X, m, n)
    op, ldo = _ptr_ld(out)
    trace = (ctypes.c_double * (max(iters, 0) + 2))()
    h.check(h.lib.qdwhg_run_fixed_iterations(h.h, m, n, X.ptr, X.ld, float(ell0), int(iters),
                                             0 if variant == "QrFirst" else 1, op, ldo, trace))
    tr = list(trace[:iters + 1])
    iq = 1 if (variant == "QrFirst" and iters > 0) else 0
    return FixedIterResult(out, tr[-1], tr, iq, iters - iq)


def _weights(w) -> float:
    return w.ell_in if isinstance(w, WeightStep) else float(w)


def qdwh_chol_step(x, w, *, handle: Optional[Handle] = None):
    """polar.hpp:56 — w: WeightStep (its ell_in is used) or ell."""
    h = handle or default_handle()
    X = _Mat(x)
    out = _empty_like_kind(X, *X.shape)
    op, ldo = _ptr_ld(out)
    h.check(h.lib.qdwhg_qdwh_chol_step(h.h, X.shape[0], X.shape[1], X.ptr, X.ld, _weights(w), op, ldo))
    return out


def qdwh_qr_step(x, w, *, handle: Optional[Handle] = None):
    """polar.hpp:53"""
    h = handle or default_handle()
    X = _Mat(x)
    out = _empty_like_kind(X, *X.shape)
    op, ldo = _ptr_ld(out)
    h.check(h.lib.qdwhg_qdwh_qr_step(h.h, X.shape[0], X.shape[1], X.ptr, X.ld, _weights(w), op, ldo))
    return out


# ------------------------------------------------------------------ kernels
def qr_factor(a, *, handle: Optional[Handle] = None):
    """kernels.hpp:18 — (Q m x m, R m x n)."""
    h = handle or default_handle()
    A = _Mat(a)
    m, n = A.shape
    Q = _empty_like_kind(A, m, m)
    R = _empty_like_kind(A, m, n)
    qp, ldq = _ptr_ld(Q)
    rp, ldr = _ptr_ld(R)
    h.check(h.lib.qdwhg_qr_factor(h.h, m, n, A.ptr, A.ld, qp, ldq, rp, ldr))
    return Q, R


def cholesky(z, *, handle: Optional[Handle] = None):
    """kernels.hpp:25 — upper W with Z = W^T W."""
    h = handle or default_handle()
    Z = _Mat(z)
    n = Z.shape[0]
    W = _empty_like_kind(Z, n, n)
    wp, ldw = _ptr_ld(W)
    h.check(h.lib.qdwhg_cholesky(h.h, n, Z.ptr, Z.ld, wp, ldw))
    return W


def sym_eig_dense(s, *, handle: Optional[Handle] = None):
    """kernels.hpp:33 — (ascending values, vectors)."""
    h = handle or default_handle()
    S = _Mat(s)
    n = S.shape[0]
    vals = np.zeros(n)
    V = _empty_like_kind(S, n, n)
    vp, ldv = _ptr_ld(V)
    h.check(h.lib.qdwhg_sym_eig_dense(h.h, n, S.ptr, S.ld, vals.ctypes.data, vp, ldv))
    return vals, V


def svd_dense(a, *, handle: Optional[Handle] = None):
    """kernels.hpp:42 — (U m x n, sigma descending, V n x n), m >= n."""
    h = handle or default_handle()
    A = _Mat(a)
    m, n = A.shape
    U = _empty_like_kind(A, m, n)
    V = _empty_like_kind(A, n, n)
    sig = np.zeros(n)
    up, ldu = _ptr_ld(U)
    vp, ldv = _ptr_ld(V)
    h.check(h.lib.qdwhg_svd_dense(h.h, m, n, A.ptr, A.ld, up, ldu, sig.ctypes.data, vp, ldv))
    return U, sig, V


@dataclass
class FullEigResult:
    """fullsolve.hpp:7-11"""
    lam: np.ndarray  # ascending
    v: object
    depth: int = 0


@dataclass
class FullSvdResult:
    """fullsolve.hpp:13-17"""
    u: object
    sigma: np.ndarray  # descending
    v: object


def qdwh_eig_full(a, base_size: int = 32, *, handle: Optional[Handle] = None) -> FullEigResult:
    """fullsolve.hpp:21 — every eigenpair by QDWH spectral divide-and-conquer."""
    h = handle or default_handle()
    A = _Mat(a)
    n = A.shape[0]
    if A.shape[1] != n:
        raise ValueError("qdwh_eig_full: matrix not square")
    lam = np.zeros(n)
    V = _empty_like_kind(A, n, n)
    vp, ldv = _ptr_ld(V)
    depth = ctypes.c_int64(0)
    h.check(h.lib.qdwhg_eig_full(h.h, n, A.ptr, A.ld, int(base_size), lam.ctypes.data, vp, ldv,
                                 ctypes.byref(depth)))
    return FullEigResult(lam=lam, v=V, depth=depth.value)


def qdwh_svd_full(a, base_size: int = 32, *, handle: Optional[Handle] = None) -> FullSvdResult:
    """fullsolve.hpp:24 — every singular triplet via the polar factor (m >= n)."""
    h = handle or default_handle()
    A = _Mat(a)
    m, n = A.shape
    U = _empty_like_kind(A, m, n)
    V = _empty_like_kind(A, n, n)
    sig = np.zeros(n)
    up, ldu = _ptr_ld(U)
    vp, ldv = _ptr_ld(V)
    h.check(h.lib.qdwhg_svd_full(h.h, m, n, A.ptr, A.ld, int(base_size), up, ldu, sig.ctypes.data,
                                 vp, ldv))
    return FullSvdResult(u=U, sigma=sig, v=V)


@dataclass
class AccuracyReport:
    """metrics.hpp:11-20"""
    orth_left: float
    orth_right: float
    value_err: Optional[float]
    resid_right: float
    resid_left: float
    n: int
    k: int


def accuracy_report(a, u, sigma, v, delta=None, paper_pairing: bool = False, *,
                    handle: Optional[Handle] = None) -> AccuracyReport:
    """metrics.hpp:25-28 (Eq. 5-7) on the device.  For a symmetric eigenreport pass
    u = v and the eigenvalues as sigma."""
    h = handle or default_handle()
    A = _Mat(a)
    m, n = A.shape
    sig = np.ascontiguousarray(np.asarray(sigma, dtype=np.float64).reshape(-1))
    k = sig.shape[0]
    dl = None if delta is None else np.ascontiguousarray(np.asarray(delta, dtype=np.float64).reshape(-1))
    if dl is not None and dl.shape[0] != k:
        raise ValueError("accuracy_report: delta length differs from sigma")
    U = _Mat(u) if k else None
    V = _Mat(v) if k else None
    if k and (U.shape[1] != k or V.shape[1] != k):
        raise ValueError("accuracy_report: sigma length must match U and V columns")
    if k and (U.shape[0] != m or V.shape[0] != n):
        raise ValueError("accuracy_report: factor shapes do not conform with A")
    out = _lib.Accuracy()
    h.check(h.lib.qdwhg_accuracy_report(
        h.h, m, n, A.ptr, A.ld, k, U.ptr if U else None, U.ld if U else 1, sig.ctypes.data,
        V.ptr if V else None, V.ld if V else 1, dl.ctypes.data if dl is not None else None,
        int(bool(paper_pairing)), ctypes.byref(out)))
    return AccuracyReport(out.orth_left, out.orth_right, out.value_err if out.has_value_err else None,
                          out.resid_right, out.resid_left, out.n, out.k)


def two_norm_estimate(a, *, handle: Optional[Handle] = None) -> float:
    """kernels.hpp:46"""
    h = handle or default_handle()
    A = _Mat(a)
    out = ctypes.c_double(0)
    h.check(h.lib.qdwhg_two_norm_estimate(h.h, A.shape[0], A.shape[1], A.ptr, A.ld,
                                          ctypes.byref(out)))
    return out.value


def lanczos_min_bound(a, steps: int = 30, *, handle: Optional[Handle] = None) -> float:
    """kernels.hpp:51"""
    h = handle or default_handle()
    A = _Mat(a)
    out = ctypes.c_double(0)
    h.check(h.lib.qdwhg_lanczos_min_bound(h.h, A.shape[0], A.ptr, A.ld, int(steps),
                                          ctypes.byref(out)))
    return out.value


KRANGE = {"full": 0, "b_upper": 1, "b_lower": 2, "a_upper": 3, "a_lower": 4}
OUTMODE = {"full": 0, "lower_mirror": 1, "lower": 2}


def gemm(a, b, c, alpha=1.0, beta=0.0, trans_a=False, trans_b=False, *, krange="full",
         out="full", diag_add=0.0, handle: Optional[Handle] = None):
    """C = alpha op(A) op(B) + beta C (+ diag_add I) on torch CUDA tensors (column-major
    views), with the triangular K-range / lower-output structure flags of qdwhg_gemm_ex."""
    h = handle or default_handle()
    A, B, C = _Mat(a), _Mat(b), _Mat(c)
    if not (A.device and B.device and C.device):
        raise ValueError("gemm: operands must be CUDA tensors")
    if C.obj is not c:
        raise ValueError("gemm: C must be a column-major view")
    m, n = C.shape
    k = A.shape[0] if trans_a else A.shape[1]
    h.check(h.lib.qdwhg_gemm_ex(h.h, int(trans_a), int(trans_b), m, n, k, float(alpha), A.ptr,
                                A.ld, B.ptr, B.ld, float(beta), C.ptr, C.ld, KRANGE[krange],
                                OUTMODE[out], float(diag_add)))
    return c


def cholesky_factor_inverse(z, *, handle: Optional[Handle] = None):
    """(W, W^{-1}), both upper, of Z = W^T W; reads the lower triangle of z
    (kernels.cpp:124-146).  Raises NotPositiveDefinite."""
    h = handle or default_handle()
    Z = _Mat(z)
    n = Z.shape[0]
    zc = Z.obj.clone() if Z.device else np.array(Z.obj, order="F", copy=True)
    Wi = _empty_like_kind(Z, n, n)
    zp, ldz = _ptr_ld(zc)
    wp, ldw = _ptr_ld(Wi)
    h.check(h.lib.qdwhg_cholesky_inverse(h.h, n, zp, ldz, wp, ldw))
    return zc, Wi


def cholesky_inverse(z, *, handle: Optional[Handle] = None):
    """W^{-1} (upper) of Z = W^T W."""
    return cholesky_factor_inverse(z, handle=handle)[1]


def cholesky_inverse_fast(z, *, handle: Optional[Handle] = None):
    """W^{-1} (upper) of a WELL-CONDITIONED Z = W^T W (the QDWH step's I + c X^T X) by
    the recursive Cholesky-and-inverse; z (lower triangle read) is not modified."""
    h = handle or default_handle()
    Z = _Mat(z)
    n = Z.shape[0]
    Wi = _empty_like_kind(Z, n, n)
    wp, ldw = _ptr_ld(Wi)
    h.check(h.lib.qdwhg_cholesky_inverse_fast(h.h, n, Z.ptr, Z.ld, wp, ldw))
    return Wi


def subspace_q2(b, tol: float = 0.01, *, handle: Optional[Handle] = None):
    """partial.cpp:71-79 — (ind, Q2): ind = first 1-based i with |R_ii| < tol of the
    unpivoted QR of b (0 if none), Q2 = Q(:, ind-1:n) (None if ind == 0)."""
    h = handle or default_handle()
    B = _Mat(b)
    n = B.shape[0]
    Q2 = _empty_like_kind(B, n, n)
    qp, ldq = _ptr_ld(Q2)
    ind = ctypes.c_int64(0)
    ell = ctypes.c_int64(0)
    h.check(h.lib.qdwhg_subspace_q2(h.h, n, B.ptr, B.ld, float(tol), ctypes.byref(ind),
                                    ctypes.byref(ell), qp, ldq, n))
    if ind.value == 0:
        return 0, None
    return int(ind.value), Q2[:, :ell.value]


def gaussian_matrix_device(m: int, n: int, seed: int, *, device=None,
                           handle: Optional[Handle] = None):
    """Counter-based N(0,1) matrix generated on the GPU (kernels.cpp:441-447 scheme)."""
    import torch
    h = handle or default_handle()
    out = torch.empty((n, m), dtype=torch.float64, device=device or "cuda").t()
    p, ld = _ptr_ld(out)
    h.check(h.lib.qdwhg_gaussian_matrix(h.h, m, n, int(seed) & (2**64 - 1), p, ld))
    return out
