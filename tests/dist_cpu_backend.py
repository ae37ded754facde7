"""TEST INFRASTRUCTURE — torch-CPU stand-in for paper_2104_14186_b200.dist.GpuBackend,
so the multi-rank orchestration (row partition, all-reduced Grams, rank-0 stages,
broadcasts) runs under gloo at world size 2 on a CPU box.  Local dense kernels
come from the CPU oracle (oracle/qdwh_oracle.py)."""
import numpy as np
import torch

from oracle import qdwh_oracle as O


class CpuBackend:
    def empty(self, m, n, like):
        return torch.empty((m, n), dtype=torch.float64)

    def empty_vec(self, n, like):
        return torch.empty(n, dtype=torch.float64)

    def from_numpy(self, a, like):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))

    def to_numpy(self, t):
        return t.numpy()

    def matmul(self, A, B, ta=False, tb=False):
        return (A.T if ta else A) @ (B.T if tb else B)

    def gram(self, X):
        return X.T @ X

    def shift_scale(self, G, c, d, symmetrize=True):
        Z = (0.5 * (G + G.T)) * c if symmetrize else G * c
        return Z + d * torch.eye(G.shape[0], dtype=G.dtype)

    def chol_factor_inv(self, Z):
        W = torch.from_numpy(O.cholesky(Z.numpy()))
        return W, torch.linalg.inv(W)

    def chol_inv(self, Z):
        return self.chol_factor_inv(Z)[1]

    def trmm_update(self, X, Winv, bc, coef):
        return bc * X + coef * ((X @ Winv) @ Winv.T)

    def zinv_update(self, X, Winv, bc, coef):
        return bc * X + coef * (X @ (Winv @ Winv.T))

    def sym_rows(self, A_full, r0, r1):
        return 0.5 * (A_full[r0:r1, :] + A_full[:, r0:r1].T)

    def shift_rows(self, A_r, a, d, r0):
        X = A_r * a
        idx = torch.arange(X.shape[0])
        X[idx, r0 + idx] += d
        return X

    def lanczos(self, A):
        return O.lanczos_min_bound(A.numpy())

    def qr_q2(self, B, tol):
        q, r = O.qr_factor(B.numpy())
        ind = O.detect_deficiency_index(r, tol)
        if ind is None:
            return 0, None
        return ind, torch.from_numpy(np.ascontiguousarray(q[:, ind - 1:]))

    def syev(self, S):
        vals, vecs = O.sym_eig_dense(S.numpy())
        return vals, torch.from_numpy(np.ascontiguousarray(vecs))

    def svd(self, R):
        u, s, v = O.svd_dense(R.numpy())
        return torch.from_numpy(np.ascontiguousarray(u)), s, torch.from_numpy(np.ascontiguousarray(v))

    def qr_step(self, X_full, w):
        return torch.from_numpy(O.qdwh_qr_step(X_full.numpy(), w))

    def gaussian(self, m, n, seed):
        return torch.from_numpy(np.ascontiguousarray(O.gaussian_matrix(m, n, seed)))

    def start_vector(self, n, seed):
        return O.gaussian_matrix(n, 1, seed)[:, 0]

    def matvec(self, A, v, trans=False):
        return (A.T @ v) if trans else (A @ v)

    def dot(self, a, b):
        return (a * b).sum().reshape(1)

    def axis(self, n, i, like):
        v = torch.zeros(n, dtype=torch.float64)
        v[i] = 1.0
        return v
