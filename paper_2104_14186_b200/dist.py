"""Multi-GPU QDWHpartial: 1D row-block distribution over ranks (one process per GPU).

The O(n^3) work of the method is the Cholesky-based QDWH steps (SURVEY.md §8(a)
a15: 80-84 % of the reference's time).  With the iterate X split by rows
(X = [X_0; X_1; ...], rank r owns X_r):

    Z = I + c * sum_r X_r^T X_r            <- local SYRK + ONE all-reduce (n x n)
    W^-1 = chol(Z)^-1                      <- replicated (n^3/3 + n^3/3)
    X_r <- (b/c) X_r + (a - b/c) X_r W^-1 W^-T   <- local TRMMs, no communication

so SYRK + both TRMMs (3 of the 3.67 n^3 per step) scale with the rank count
and the only data-path collective is the Gram all-reduce (the paper's
2D block-cyclic ScaLAPACK layout, is the next refinement).
The remaining O(n^3) stages are much smaller and run on rank 0 with the
result broadcast: the subspace QR and Q2 (partial.cpp:71-79 / 138-146), the
ell x ell Rayleigh-Ritz EIG/SVD; distributed products are used where they are
natural (A Q2 by rows, Q2^T (A Q2) by an all-reduce of ell x ell partials,
the tall-skinny CholeskyQR2 of A Q2 by all-reduced Grams).  Lanczos and the
power-iteration norm (HBM-bound scalars) follow the reference control flow
with all-reduced dot products, so every rank takes identical decisions.

Backends: `GpuBackend` runs every local op in libqdwhg (torch CUDA tensors,
NCCL collectives); tests/dist_cpu_backend.py provides a torch-CPU stand-in so
the orchestration is exercised with gloo at world size 2 on a CPU box.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

EPS = float(np.finfo(np.float64).eps)


def row_range(m: int, rank: int, world: int):
    """Balanced contiguous row block of rank (rows [r0, r1))."""
    base, extra = divmod(m, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


class Comm:
    """torch.distributed wrapper (NCCL on GPU, gloo on CPU)."""

    def __init__(self, dist, group=None):
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    @staticmethod
    def _dense(t):
        """A contiguous alias of t's storage (column-major views are row-major transposes)."""
        if t.is_contiguous():
            return t
        if t.dim() == 2 and t.t().is_contiguous():
            return t.t()
        return None

    def allreduce(self, t):
        x = self._dense(t)
        if x is None:
            x = t.contiguous()
            self.dist.all_reduce(x, group=self.group)
            t.copy_(x)
        else:
            self.dist.all_reduce(x, group=self.group)
        return t

    def broadcast(self, t, src=0):
        x = self._dense(t)
        if x is None:
            x = t.contiguous()
            self.dist.broadcast(x, src=src, group=self.group)
            t.copy_(x)
        else:
            self.dist.broadcast(x, src=src, group=self.group)
        return t

    def allgather_rows(self, t, m):
        """Concatenate the row blocks of all ranks (balanced split of m rows)."""
        import torch
        parts = []
        for r in range(self.world):
            r0, r1 = row_range(m, r, self.world)
            parts.append(torch.empty((r1 - r0, t.shape[1]), dtype=t.dtype, device=t.device))
        self.dist.all_gather(parts, t.contiguous(), group=self.group)
        return torch.cat(parts, dim=0)

    def bcast_scalar(self, x: float, like):
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=like.device)
        self.broadcast(t)
        return float(t.item())


@dataclass
class DistResult:
    values: np.ndarray
    v: object          # replicated n x k (EIG) or V1 (SVD)
    u_rows: object = None  # SVD: this rank's rows of U1
    subspace_size: int = 0
    rank_index: int = 0
    scale: float = 0.0     # mu (EIG) or alpha (SVD)
    iters_chol: int = 0
    iters_qr: int = 0
    ell_trace: list = field(default_factory=list)
    flops: float = 0.0


def halley(ell):
    from . import qdwh
    return qdwh.halley_weights(ell)


def _chol_step_rows(be, comm, X_r, w, symmetric=False):
    """One Cholesky-based QDWH step on row-distributed X (polar.cpp:82-128).
    symmetric (EIG path): X Z^{-1} with the replicated Z^{-1} = W^{-1} W^{-T} (one
    LAUUM + one local GEMM: 4/3 n^3 instead of the two TRMMs' 5/3 n^3)."""
    G = be.gram(X_r)                       # X_r^T X_r
    comm.allreduce(G)                      # sum over ranks
    Z = be.shift_scale(G, w.c, 1.0)        # I + c * sym(G)
    Winv = be.chol_inv(Z)                  # replicated, throws NotPositiveDefinite
    bc = w.b / w.c
    if symmetric:
        return be.zinv_update(X_r, Winv, bc, w.a - bc)
    return be.trmm_update(X_r, Winv, bc, w.a - bc)


def dist_partial_eig(be, comm, A_r, n: int, s: float = 0.2, iters: int = 3, tol: float = 0.01,
                     randomize: bool = False, seed: int = 0) -> DistResult:
    """Alg. 1 (partial.cpp:40-99) with A given by rows: A_r = A[r0:r1, :] (symmetric A)."""
    r0, r1 = row_range(n, comm.rank, comm.world)
    A_full = comm.allgather_rows(A_r, n)   # needed for the symmetry check / Lanczos on rank 0
    res = DistResult(values=np.zeros(0), v=None)
    mu = be.lanczos(A_full) if comm.rank == 0 else 0.0
    mu = comm.bcast_scalar(mu, A_r)
    res.scale = mu
    if mu >= 0.0:
        return res
    scale = abs(mu)
    As_r = be.sym_rows(A_full, r0, r1) * (1.0 / scale)   # rows of sym(A)/|mu|
    X_r = be.shift_rows(As_r, 1.0 - s, -s, r0)           # (1-s) As - s I, own rows
    ell = s
    res.ell_trace = [ell]
    for _ in range(iters):
        w = halley(ell)
        X_r = _chol_step_rows(be, comm, X_r, w, symmetric=True)
        X_full = comm.allgather_rows(X_r, n)             # symmetrize (polar.cpp:210)
        X_r = be.sym_rows(X_full, r0, r1)
        res.iters_chol += 1
        ell = w.ell_out
        res.ell_trace.append(ell)
    X_full = comm.allgather_rows(X_r, n)
    # subspace extraction and Rayleigh-Ritz on rank 0, broadcast
    if comm.rank == 0:
        B = be.shift_scale(X_full, 0.5, 0.5, symmetrize=False)  # (X + I)/2
        if randomize:
            B = be.matmul(B, be.gaussian(n, n, seed))
        ind, Q2 = be.qr_q2(B, tol)
    else:
        ind, Q2 = 0, None
    ind = int(comm.bcast_scalar(float(ind), A_r))
    res.rank_index = ind
    if ind == 0:
        return res
    ellw = n - ind + 1
    res.subspace_size = ellw
    if Q2 is None:
        Q2 = be.empty(n, ellw, like=A_r)
    comm.broadcast(Q2)
    AQ_r = be.matmul(As_r, Q2)                           # rows r of (A/|mu|) Q2
    S = be.matmul(Q2[r0:r1], AQ_r, ta=True)              # partial Q2^T A Q2
    comm.allreduce(S)
    S = 0.5 * (S + S.T)
    if comm.rank == 0:
        vals, W = be.syev(S)
        vals_t = be.from_numpy(vals, like=A_r)
    else:
        vals_t, W = be.empty_vec(ellw, like=A_r), be.empty(ellw, ellw, like=A_r)
    comm.broadcast(vals_t)
    comm.broadcast(W)
    vals = be.to_numpy(vals_t)
    k = 0
    while k < ellw and vals[k] < 0.0:
        k += 1
    res.values = scale * vals[:k]
    res.v = be.matmul(Q2, W[:, :k]) if k else None
    nd, l = float(n), float(ellw)
    res.flops = (iters * 10.0 / 3.0 * nd ** 3 + 4.0 / 3.0 * nd ** 3 + 4 * nd * nd * l
                 - 2 * l ** 3 / 3 + 2 * nd * l * l + 9 * l ** 3 + 2 * nd * l * k)
    return res


def dist_two_norm(be, comm, A_r, n):
    """kernels.cpp:332-360 with all-reduced products (identical decisions on all ranks)."""
    from . import qdwh  # noqa: F401
    v = be.from_numpy(be.start_vector(n, 0x6E6F726D32), like=A_r)
    est = 0.0
    for it in range(100):
        y_r = be.matvec(A_r, v)
        ny2 = comm.allreduce(be.dot(y_r, y_r))
        ny = math.sqrt(float(ny2.item()))
        if ny == 0.0:
            v = be.axis(n, it % n, like=A_r)
            continue
        z = comm.allreduce(be.matvec(A_r, y_r, trans=True))
        nz = math.sqrt(float(be.dot(z, z).item()))
        prev, est = est, ny
        if nz == 0.0:
            break
        v = z / nz
        if it > 0 and abs(est - prev) < 1e-3 * est:
            break
    return 1.05 * est


def dist_partial_svd(be, comm, A_r, m: int, n: int, s: float = None, cut: float = None,
                     tol: float = 0.01, randomize: bool = False, seed: int = 0) -> DistResult:
    """Alg. 2 (partial.cpp:101-158) with A given by rows; s relative or an absolute cut."""
    from . import qdwh
    r0, r1 = row_range(m, comm.rank, comm.world)
    res = DistResult(values=np.zeros(0), v=None)
    alpha = dist_two_norm(be, comm, A_r, n)
    res.scale = alpha
    if cut is not None:
        s = cut / alpha
    if not (s > 0.0) or s >= 1.0:
        raise ValueError("qdwh_partial_svd: threshold s must be in (0, 1)")
    X_r = A_r * (1.0 / alpha)
    iters = qdwh.iterations_to_converge(s, 5.0 * EPS)
    ell = s
    res.ell_trace = [ell]
    for k in range(iters):
        w = halley(ell)
        if s < 1e-3 and k == 0:
            X_full = comm.allgather_rows(X_r, m)             # QR step replicated
            X_r = be.qr_step(X_full, w)[r0:r1]
            res.iters_qr += 1
        else:
            X_r = _chol_step_rows(be, comm, X_r, w)
            res.iters_chol += 1
        ell = w.ell_out
        res.ell_trace.append(ell)
    G = comm.allreduce(be.gram(X_r))
    if comm.rank == 0:
        M = be.shift_scale(G, -1.0, 1.0)                     # I - sym(X^T X)
        if randomize:
            M = be.matmul(M, be.gaussian(n, n, seed))
        ind, Q2 = be.qr_q2(M, tol)
    else:
        ind, Q2 = 0, None
    ind = int(comm.bcast_scalar(float(ind), A_r))
    res.rank_index = ind
    if ind == 0:
        return res
    ellw = n - ind + 1
    res.subspace_size = ellw
    if Q2 is None:
        Q2 = be.empty(n, ellw, like=A_r)
    comm.broadcast(Q2)
    Y_r = be.matmul(A_r, Q2)                                 # rows of A Q2 (unscaled A)
    # tall-skinny CholeskyQR2 with all-reduced Grams: Y = Q R.  Every rank holds
    # the same reduced Grams, so the success test is taken identically everywhere.
    from .qdwh import NotPositiveDefinite
    ok = True
    try:
        G1 = comm.allreduce(be.gram(Y_r))
        W1, W1inv = be.chol_factor_inv(G1)
        d = np.abs(np.diagonal(be.to_numpy(W1)))
        # R from the Grams perturbs sigma_i^2 by ~u*sigma_max^2: keep the Gram route
        # only while that stays far inside the 1e-10 relative gate (kappa <~ 1e2)
        ok = bool(d.min() > 0.0 and d.max() / d.min() <= 1e2)
        if ok:
            Q1_r = be.matmul(Y_r, W1inv)
            G2 = comm.allreduce(be.gram(Q1_r))
            W2, W2inv = be.chol_factor_inv(G2)
            Q_r = be.matmul(Q1_r, W2inv)
    except RuntimeError as e:  # qdwh.NotPositiveDefinite (GPU) / oracle's (CPU stand-in)
        if type(e).__name__ != NotPositiveDefinite.__name__:
            raise
        ok = False
    if not ok:
        # ill-conditioned A Q2: Householder SVD of the gathered Y on rank 0
        Y = comm.allgather_rows(Y_r, m)
        if comm.rank == 0:
            U, sig, VR = be.svd(Y)
            sig_t = be.from_numpy(sig, like=A_r)
        else:
            U, VR = be.empty(m, ellw, like=A_r), be.empty(ellw, ellw, like=A_r)
            sig_t = be.empty_vec(ellw, like=A_r)
        for t in (U, sig_t, VR):
            comm.broadcast(t)
        Q_r, UR = U[r0:r1], None
    if ok and comm.rank == 0:
        R = be.matmul(W2, W1)                                # R = W2 W1 (upper)
        UR, sig, VR = be.svd(R)
        sig_t = be.from_numpy(sig, like=A_r)
    elif ok:
        UR, VR = be.empty(ellw, ellw, like=A_r), be.empty(ellw, ellw, like=A_r)
        sig_t = be.empty_vec(ellw, like=A_r)
    if ok:
        for t in (UR, sig_t, VR):
            comm.broadcast(t)
    sig = be.to_numpy(sig_t)
    cutoff = s * alpha
    k = 0
    while k < len(sig) and sig[k] > cutoff:
        k += 1
    res.values = sig[:k]
    if k:
        res.u_rows = be.matmul(Q_r, UR[:, :k]) if ok else Q_r[:, :k]
        res.v = be.matmul(Q2, VR[:, :k])
    md, nd, l = float(m), float(n), float(ellw)
    res.flops = (res.iters_qr * (6 * md * nd * nd + 8.0 / 3.0 * nd ** 3)
                 + res.iters_chol * (3 * md * nd * nd + nd ** 3 / 3) + md * nd * nd
                 + 4.0 / 3.0 * nd ** 3 + 2 * nd * nd * l - 2 * l ** 3 / 3 + 2 * md * nd * l
                 + 6 * md * l * l + 20 * l ** 3 + 2 * nd * l * k)
    return res


class GpuBackend:
    """Local ops on torch CUDA tensors through libqdwhg (no cuBLAS/cuSOLVER)."""

    def __init__(self, handle):
        from . import qdwh
        self.q = qdwh
        self.h = handle

    @staticmethod
    def _cm(t):
        return t.t().contiguous().t()

    def empty(self, m, n, like):
        import torch
        return torch.empty((n, m), dtype=torch.float64, device=like.device).t()

    def empty_vec(self, n, like):
        import torch
        return torch.empty(n, dtype=torch.float64, device=like.device)

    def from_numpy(self, a, like):
        import torch
        return torch.from_numpy(np.ascontiguousarray(a)).to(like.device)

    def to_numpy(self, t):
        return t.detach().cpu().numpy()

    def matmul(self, A, B, ta=False, tb=False):
        m = A.shape[1] if ta else A.shape[0]
        n = B.shape[0] if tb else B.shape[1]
        C = self.empty(m, n, like=A)
        return self.q.gemm(self._cm(A), self._cm(B), C, trans_a=ta, trans_b=tb, handle=self.h)

    def gram(self, X):
        n = X.shape[1]
        C = self.empty(n, n, like=X)
        return self.q.gemm(self._cm(X), self._cm(X), C, trans_a=True, out="lower_mirror",
                           handle=self.h)

    def shift_scale(self, G, c, d, symmetrize=True):
        import torch
        Z = (0.5 * (G + G.T)) * c if symmetrize else G * c
        Z = Z + d * torch.eye(G.shape[0], dtype=G.dtype, device=G.device)
        return self._cm(Z)

    def chol_inv(self, Z):
        # kappa(Z) <= 1 + c in the QDWH step: the recursive Cholesky-and-inverse
        return self.q.cholesky_inverse_fast(self._cm(Z), handle=self.h)

    def zinv_update(self, X, Winv, bc, coef):
        """(b/c) X + (a - b/c) X Z^{-1}, Z^{-1} = W^{-1} W^{-T} (LAUUM: lower tiles,
        K from the tile row, mirrored)."""
        n = Winv.shape[0]
        Winv = self._cm(Winv)
        WiT = self._cm(Winv.T)
        Zi = self.empty(n, n, like=X)
        self.q.gemm(Winv, WiT, Zi, krange="a_upper", out="lower_mirror", handle=self.h)
        Xo = self._cm(X.clone())
        return self.q.gemm(self._cm(X), Zi, Xo, alpha=coef, beta=bc, handle=self.h)

    def trmm_update(self, X, Winv, bc, coef):
        Y = self.empty(X.shape[0], X.shape[1], like=X)
        self.q.gemm(self._cm(X), Winv, Y, krange="b_upper", handle=self.h)
        Xo = self._cm(X.clone())
        return self.q.gemm(Y, Winv, Xo, alpha=coef, beta=bc, trans_b=True, krange="b_lower",
                           handle=self.h)

    def sym_rows(self, A_full, r0, r1):
        return self._cm(0.5 * (A_full[r0:r1, :] + A_full[:, r0:r1].T))

    def shift_rows(self, A_r, a, d, r0):
        X = A_r * a
        idx = np.arange(X.shape[0])
        X[idx, r0 + idx] += d
        return self._cm(X)

    def lanczos(self, A):
        return self.q.lanczos_min_bound(self._cm(A), handle=self.h)

    def qr_q2(self, B, tol):
        # partial.cpp:71-79 on the device: trailing-column Q formation only
        ind, Q2 = self.q.subspace_q2(self._cm(B), tol, handle=self.h)
        return ind, (self._cm(Q2) if Q2 is not None else None)

    def syev(self, S):
        vals, V = self.q.sym_eig_dense(self._cm(S), handle=self.h)
        return vals, V

    def svd(self, R):
        U, s, V = self.q.svd_dense(self._cm(R), handle=self.h)
        return U, s, V

    def chol_factor_inv(self, Z):
        """(W, W^-1) with Z = W^T W."""
        W, Winv = self.q.cholesky_factor_inverse(self._cm(Z), handle=self.h)
        return W, Winv

    def qr_step(self, X_full, w):
        return self.q.qdwh_qr_step(self._cm(X_full), w.ell_in, handle=self.h)

    def gaussian(self, m, n, seed):
        return self.q.gaussian_matrix_device(m, n, seed, handle=self.h)

    def start_vector(self, n, seed):
        from .matgen import gaussian_host
        return gaussian_host(n, seed)

    def matvec(self, A, v, trans=False):
        # GEMV through the DMMA engine (HBM-bound; keeps cuBLAS off the path)
        vm = v.reshape(-1, 1)
        out = self.empty(A.shape[1] if trans else A.shape[0], 1, like=A)
        self.q.gemm(self._cm(A), self._cm(vm), out, trans_a=trans, handle=self.h)
        return out.reshape(-1)

    def dot(self, a, b):
        return (a * b).sum().reshape(1)

    def axis(self, n, i, like):
        import torch
        v = torch.zeros(n, dtype=torch.float64, device=like.device)
        v[i] = 1.0
        return v
