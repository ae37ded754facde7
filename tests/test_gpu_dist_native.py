"""The C++ distributed driver (libqdwhg qdwhg_dist_*) on the GPU.

Only one B200 is available to the test runner, so the multi-rank path runs as
emulated ranks: one thread per rank, each with its own qdwhg handle (stream,
arena) on cuda:0, over the in-process loopback communicator — the engine is
the real sm_100a one (DMMA GEMMs, Cholesky-and-inverse leaves, register panel
QR, device Rayleigh-Ritz).  No kernel waits on another rank (collectives are
host rendezvous + copies), so this is safe on one GPU.  The NCCL communicator
itself runs at world size 1 (1 x 1 grid)."""
import threading

import numpy as np
import pytest

from oracle import qdwh_oracle as O
from paper_2104_14186_b200 import matgen, qdwh

pytestmark = pytest.mark.gpu


def run_grid(P, Q, nb, body):
    world = qdwh.LoopbackWorld(P * Q)
    out, errs = [None] * (P * Q), [None] * (P * Q)

    def rank(r):
        try:
            h = qdwh.Handle(device=0)
            d = qdwh.Dist(h, P, Q, nb, r, world=world)
            out[r] = body(d, r)
            d.close()
            h.close()
        except Exception as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=rank, args=(r,)) for r in range(P * Q)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    world.close()
    for e in errs:
        if e is not None:
            raise e
    return out


@pytest.mark.parametrize("P,Q", [(1, 2), (2, 1), (2, 2)])
@pytest.mark.parametrize("ta,tb,flags", [(0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0), (0, 0, 1), (0, 0, 4),
                                         (0, 1, 1 | 8 | 16), (1, 0, 16)])
def test_emulated_pgemm(P, Q, ta, tb, flags):
    rng = np.random.default_rng(7)
    n, nb = 1536, 256
    U = np.triu(rng.standard_normal((n, n)))
    X = rng.standard_normal((n, n))
    A = U if flags & 1 else X
    B = U if flags & 4 or flags & 8 else rng.standard_normal((n, n))
    C0 = rng.standard_normal((n, n))
    res = run_grid(P, Q, nb, lambda d, r: d.pgemm(A, B, C0, 0.5, -1.0, ta, tb, flags))
    want = 0.5 * (A.T if ta else A) @ (B.T if tb else B) - C0
    got = res[0]
    if flags & 16:
        tl = np.kron(np.tril(np.ones((n // nb, n // nb))), np.ones((nb, nb))).astype(bool)
        np.testing.assert_allclose(got[tl], want[tl], rtol=1e-10, atol=1e-10)
    else:
        np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-10)


@pytest.mark.parametrize("P,Q", [(1, 2), (2, 1), (2, 2)])
def test_emulated_chol_inv_and_qr(P, Q):
    rng = np.random.default_rng(11)
    n, nb = 1536, 256
    X = rng.standard_normal((n, n)) / np.sqrt(n)
    Z = np.eye(n) + 3.0 * X.T @ X
    res = run_grid(P, Q, nb, lambda d, r: d.cholesky_inverse(Z))
    W = np.linalg.cholesky(Z).T
    np.testing.assert_allclose(res[0], np.linalg.inv(W), rtol=1e-9, atol=1e-11)
    c0, ell = 1000, 536
    res = run_grid(P, Q, nb, lambda d, r: d.qr(X, c0, ell))
    q, r = np.linalg.qr(X, mode="complete")
    for rd, _ in res:
        np.testing.assert_allclose(rd, np.abs(np.diag(r)), rtol=1e-9)
    q2 = res[0][1]
    np.testing.assert_allclose(np.abs(q2), np.abs(q[:, c0:c0 + ell]), atol=1e-10)


def planted(n, family, k, seed=42):
    lam = matgen.config_eigenvalues(family, n, seed)
    q, _ = np.linalg.qr(O.gaussian_matrix(n, n, seed))
    a = (q * lam) @ q.T
    return np.asfortranarray(0.5 * (a + a.T)), lam, matgen.largest_k_shift(lam, k)


@pytest.mark.parametrize("P,Q,nb", [(1, 2, 256), (2, 2, 256), (2, 1, 128)])
def test_emulated_grid_partial_eig(P, Q, nb):
    n, k = 1536, 15
    a, lam, c = planted(n, "logsigned", k)
    res = run_grid(P, Q, nb, lambda d, r: d.partial_eig_request(a, "largest", c, k))
    r0 = res[0]
    assert r0.count() == k
    want = np.sort(lam)[::-1][:k]
    np.testing.assert_allclose(r0.lambda_minus, want, rtol=1e-10, atol=1e-14)
    for r in res[1:]:  # values replicated on every rank
        np.testing.assert_allclose(r.lambda_minus, r0.lambda_minus, rtol=0, atol=0)
    single = qdwh.partial_eig_request(a, "largest", c, k)
    np.testing.assert_allclose(r0.lambda_minus, single.lambda_minus, rtol=1e-12)
    assert r0.subspace_size == single.subspace_size
    v = np.asarray(r0.v)
    resid = np.linalg.norm(a @ v - v * r0.lambda_minus) / np.linalg.norm(a)
    orth = np.linalg.norm(np.eye(k) - v.T @ v)
    assert resid <= 1e-12 * np.sqrt(n) and orth <= 1e-12 * np.sqrt(n), (resid, orth)


def test_emulated_grid_partial_svd_device_resident(cuda):
    import torch
    m, n, k = 2048, 1024, 60
    sig = matgen.config_singular_values("inv", n)
    ul, _ = np.linalg.qr(O.gaussian_matrix(m, n, 42 ^ matgen.LEFT_STREAM))
    vr, _ = np.linalg.qr(O.gaussian_matrix(n, n, 42 ^ matgen.RIGHT_STREAM))
    a = np.asfortranarray((ul * sig) @ vr.T)
    at = torch.from_numpy(a).to(cuda).t().contiguous().t()
    cut = matgen.sigma_cut(sig, k)

    def body(d, r):
        d.load(at)
        return d.partial_svd_request(None, cut=cut, k=k, use_randomization=True, seed=5)

    res = run_grid(2, 2, 256, body)
    r0 = res[0]
    assert r0.count() == k
    np.testing.assert_allclose(r0.sigma1, sig[:k], rtol=1e-10)
    u, v = r0.u1, r0.v1
    s = torch.from_numpy(np.asarray(r0.sigma1)).to(cuda)
    assert float(torch.linalg.norm(at @ v - u * s[None, :]) / torch.linalg.norm(at)) <= 1e-12 * np.sqrt(n)
    eye = torch.eye(k, dtype=torch.float64, device=cuda)
    assert float(torch.linalg.norm(eye - v.T @ v)) <= 1e-12 * np.sqrt(n)
    assert float(torch.linalg.norm(eye - u.T @ u)) <= 1e-12 * np.sqrt(n)


def test_nccl_world_of_one():
    """The NCCL communicator (ncclCommInitRank + row/column ncclCommSplit,
    broadcasts, all-reductions, send/recv) at world size 1."""
    n, k = 1024, 10
    a, lam, c = planted(n, "uniform", k)
    h = qdwh.Handle(device=0)
    d = qdwh.Dist(h, 1, 1, 256, 0, unique_id=qdwh.dist_unique_id())
    r = d.partial_eig_request(a, "largest", c, k)
    assert r.count() == k
    np.testing.assert_allclose(r.lambda_minus, np.sort(lam)[::-1][:k], rtol=1e-10)
    assert d.stats()["collectives"] > 0
    d.close()
