"""The distributed 2D block-cyclic driver (paper_2104_14186_b200/csrc/dist/,
compiled unchanged) on CPU: emulated ranks as threads over the loopback
communicator and a plain host engine (tests/cpp/dist_host.cpp, test-only).
World sizes 2 (1x2, 2x1) and 4 (2x2), tile sizes that leave partial edge tiles,
checked against numpy (building blocks) and the pinned oracle (drivers)."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

from oracle import qdwh_oracle as O
from paper_2104_14186_b200 import matgen

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "cpp", "libqdwhg_disthost.so")
GRIDS = [(1, 2), (2, 1), (2, 2)]
P_ = ctypes.c_void_p
I64 = ctypes.c_int64
D = ctypes.c_double
I = ctypes.c_int


@pytest.fixture(scope="module")
def dh():
    subprocess.check_call(["make", "-s", "-C", os.path.join(HERE, "cpp")])
    lib = ctypes.CDLL(LIB)
    lib.dh_pgemm.argtypes = [I, I, I, I, I, I64, I64, I64, D, P_, I64, P_, I64, D, P_, P_, I64, I, P_, I]
    lib.dh_chol_inv.argtypes = [I, I, I, I64, P_, I64, P_, I64, P_, I]
    lib.dh_qr.argtypes = [I, I, I, I64, I64, P_, I64, I64, I64, P_, P_, I64, P_, I]
    lib.dh_partial_eig.argtypes = [I, I, I, I64, P_, I64, D, I64, I, ctypes.c_uint64, P_, P_, I64, P_, P_, P_,
                                   P_, I]
    lib.dh_partial_svd.argtypes = [I, I, I, I64, I64, P_, I64, D, I64, I, ctypes.c_uint64, P_, P_, I64, P_, I64,
                                   P_, P_, P_, P_, I]
    return lib


def F(a):
    return np.asfortranarray(a, dtype=np.float64)


def p(a):
    return a.ctypes.data_as(P_)


def check(rc, err):
    assert rc == 0, err.value.decode()


@pytest.mark.parametrize("grid", GRIDS)
@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_pgemm_transposes(dh, grid, ta, tb):
    rng = np.random.default_rng(3)
    m, n, k, nb = 100, 70, 90, 32
    A = F(rng.standard_normal((k, m) if ta else (m, k)))
    B = F(rng.standard_normal((n, k) if tb else (k, n)))
    C = F(rng.standard_normal((m, n)))
    out = F(np.zeros((m, n)))
    err = ctypes.create_string_buffer(512)
    check(dh.dh_pgemm(*grid, nb, ta, tb, m, n, k, 0.7, p(A), A.shape[0], p(B), B.shape[0], -0.3, p(C), p(out),
                      m, 0, err, 512), err)
    want = 0.7 * (A.T if ta else A) @ (B.T if tb else B) - 0.3 * C
    np.testing.assert_allclose(out, want, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("grid", GRIDS)
def test_pgemm_structure_flags(dh, grid):
    """Triangular operands skip their zero tiles (results equal the dense
    product) and c_lower computes only the lower tiles."""
    rng = np.random.default_rng(5)
    n, nb = 160, 32
    U = F(np.triu(rng.standard_normal((n, n))))
    L = F(np.tril(rng.standard_normal((n, n))))
    X = F(rng.standard_normal((n, n)))
    err = ctypes.create_string_buffer(512)
    cases = [(U, X, 0, 0, 1, U @ X), (L, X, 0, 0, 2, L @ X), (X, U, 0, 0, 4, X @ U), (X, L, 0, 0, 8, X @ L),
             (U, U, 0, 1, 1 | 8 | 16, U @ U.T), (U, L, 1, 1, 2 | 4, U.T @ L.T)]
    for A, B, ta, tb, flags, want in cases:
        C0 = F(np.full((n, n), 7.0))
        out = F(np.zeros((n, n)))
        check(dh.dh_pgemm(*grid, nb, ta, tb, n, n, n, 1.0, p(A), n, p(B), n, 0.0, p(C0), p(out), n, flags, err,
                          512), err)
        if flags & 16:  # lower tiles computed, upper tiles untouched (7.0)
            tl = np.kron(np.tril(np.ones((n // nb, n // nb))), np.ones((nb, nb))).astype(bool)
            np.testing.assert_allclose(out[tl], want[tl], rtol=1e-11, atol=1e-11)
            assert np.all(out[~tl] == 7.0)
        else:
            np.testing.assert_allclose(out, want, rtol=1e-11, atol=1e-11)


@pytest.mark.parametrize("grid", GRIDS + [(1, 1)])
@pytest.mark.parametrize("n,nb", [(96, 32), (150, 32), (256, 64)])
def test_chol_inv(dh, grid, n, nb):
    rng = np.random.default_rng(n)
    X = rng.standard_normal((n, n)) / np.sqrt(n)
    Z = F(np.eye(n) + 3.0 * X.T @ X)  # kappa ~ the QDWH steps'
    Zl = F(np.tril(Z) + np.triu(np.full((n, n), np.nan), 1))  # only the lower triangle is read
    Wi = F(np.zeros((n, n)))
    err = ctypes.create_string_buffer(512)
    check(dh.dh_chol_inv(*grid, nb, n, p(Zl), n, p(Wi), n, err, 512), err)
    W = np.linalg.cholesky(Z).T
    np.testing.assert_allclose(Wi, np.linalg.inv(W), rtol=1e-10, atol=1e-12)
    assert np.all(np.tril(Wi, -1) == 0.0)


def test_chol_inv_not_positive_definite_on_every_rank(dh):
    n = 96
    Z = F(np.diag(np.r_[np.ones(70), -1.0, np.ones(25)]))
    Wi = F(np.zeros((n, n)))
    err = ctypes.create_string_buffer(512)
    rc = dh.dh_chol_inv(2, 2, 32, n, p(Z), n, p(Wi), n, err, 512)
    assert rc != 0 and b"pivot" in err.value


@pytest.mark.parametrize("grid", GRIDS)
@pytest.mark.parametrize("m,n,nb", [(128, 128, 32), (150, 110, 32), (192, 192, 64)])
def test_qr_rdiag_and_trailing_q(dh, grid, m, n, nb):
    rng = np.random.default_rng(m + n)
    X = F(rng.standard_normal((m, n)))
    c0 = n // 3
    ell = m - c0
    rd = np.zeros(n)
    Q2 = F(np.zeros((m, ell)))
    err = ctypes.create_string_buffer(512)
    check(dh.dh_qr(*grid, nb, m, n, p(X), m, c0, ell, p(rd), p(Q2), m, err, 512), err)
    q, r = np.linalg.qr(X, mode="complete")
    np.testing.assert_allclose(rd, np.abs(np.diag(r)), rtol=1e-11)
    # same columns of Q up to sign (LAPACK and the reference share the reflector convention)
    np.testing.assert_allclose(np.abs(Q2), np.abs(q[:, c0:c0 + ell]), atol=1e-11)
    np.testing.assert_allclose(Q2.T @ Q2, np.eye(ell), atol=1e-12)


def sym_planted(n, lam, seed):
    q, _ = np.linalg.qr(O.gaussian_matrix(n, n, seed))
    a = (q * lam) @ q.T
    return F(0.5 * (a + a.T))


@pytest.mark.parametrize("grid", GRIDS + [(1, 1)])
@pytest.mark.parametrize("n,nb,family,k", [(192, 32, "uniform", 19), (200, 64, "logsigned", 6)])
def test_dist_partial_eig_vs_oracle(dh, grid, n, nb, family, k):
    lam = matgen.config_eigenvalues(family, n, 42)
    a = sym_planted(n, lam, 42)
    c = matgen.largest_k_shift(lam, k)
    vals = np.zeros(n)
    V = F(np.zeros((n, n)))
    ko, ello, mu = I64(0), I64(0), D(0)
    err = ctypes.create_string_buffer(512)
    check(dh.dh_partial_eig(*grid, nb, n, p(a), n, c, k, 0, 0, p(vals), p(V), n, ctypes.byref(ko),
                            ctypes.byref(ello), ctypes.byref(mu), err, 512), err)
    ref = O.qdwh_partial_eig(c * np.eye(n) - a, O.choose_shift(3))
    assert ko.value == k and ref.count() == k
    np.testing.assert_allclose(vals[:k], c - ref.lambda_minus[:k], rtol=1e-10)
    np.testing.assert_allclose(mu.value, ref.mu, rtol=1e-10)
    assert ello.value == ref.subspace_size
    v = V[:, :k]
    res = np.linalg.norm(a @ v - v * vals[:k]) / np.linalg.norm(a)
    orth = np.linalg.norm(np.eye(k) - v.T @ v)
    assert res <= 1e-12 * np.sqrt(n) and orth <= 1e-12 * np.sqrt(n), (res, orth)


def test_dist_partial_eig_randomized_wishart(dh):
    n, nb, k = 160, 32, 32
    g = O.gaussian_matrix(n, n, 42)
    a = F(0.5 * ((g.T @ g / n - np.eye(n)) + (g.T @ g / n - np.eye(n)).T))
    w = np.sort(np.linalg.eigvalsh(a))[::-1]
    c = matgen.CONFIGS[4]["shift"]
    vals = np.zeros(n)
    V = F(np.zeros((n, n)))
    ko, ello, mu = I64(0), I64(0), D(0)
    err = ctypes.create_string_buffer(512)
    check(dh.dh_partial_eig(2, 2, nb, n, p(a), n, c, k, 1, 7, p(vals), p(V), n, ctypes.byref(ko),
                            ctypes.byref(ello), ctypes.byref(mu), err, 512), err)
    assert ko.value == k
    np.testing.assert_allclose(vals[:k], w[:k], rtol=1e-10)


@pytest.mark.parametrize("grid", GRIDS)
@pytest.mark.parametrize("m,n,nb,k,rnd", [(160, 160, 32, 16, 0), (224, 96, 32, 10, 1)])
def test_dist_partial_svd_vs_oracle(dh, grid, m, n, nb, k, rnd):
    sig = matgen.config_singular_values("log16" if m == n else "inv", n)
    ul, _ = np.linalg.qr(O.gaussian_matrix(m, n, 42 ^ matgen.LEFT_STREAM))
    vr, _ = np.linalg.qr(O.gaussian_matrix(n, n, 42 ^ matgen.RIGHT_STREAM))
    a = F((ul * sig) @ vr.T)
    cut = matgen.sigma_cut(sig, k)
    s = np.zeros(n)
    U = F(np.zeros((m, n)))
    V = F(np.zeros((n, n)))
    ko, ello, al = I64(0), I64(0), D(0)
    err = ctypes.create_string_buffer(512)
    check(dh.dh_partial_svd(*grid, nb, m, n, p(a), m, cut, k, rnd, 3, p(s), p(U), m, p(V), n, ctypes.byref(ko),
                            ctypes.byref(ello), ctypes.byref(al), err, 512), err)
    alpha = O.two_norm_estimate(a)
    ref = O.qdwh_partial_svd(a, cut / alpha, use_randomization=bool(rnd), seed=3)
    assert ko.value == k and ref.count() == k
    np.testing.assert_allclose(al.value, alpha, rtol=1e-12)
    np.testing.assert_allclose(s[:k], ref.sigma1[:k], rtol=1e-10)
    np.testing.assert_allclose(s[:k], sig[:k], rtol=1e-10)
    u, v = U[:, :k], V[:, :k]
    assert np.linalg.norm(a @ v - u * s[:k]) / np.linalg.norm(a) <= 1e-12 * np.sqrt(n)
    assert np.linalg.norm(np.eye(k) - v.T @ v) <= 1e-12 * np.sqrt(n)
    assert np.linalg.norm(np.eye(k) - u.T @ u) <= 1e-12 * np.sqrt(n)
