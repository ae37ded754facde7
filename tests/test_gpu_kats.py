"""The reference's known-answer tests for the polar / fixed-iteration / partial
drivers, re-expressed against libqdwhg through the C ABI.
Inputs are built with numpy from the oracle's seeded Gaussian generator; each
test cites the reference test it restates.  Marked gpu."""
import numpy as np
import pytest

from oracle import qdwh_oracle as O
from paper_2104_14186_b200 import qdwh

pytestmark = pytest.mark.gpu
U = O.EPS


def orthogonal(n, seed):
    q, r = np.linalg.qr(O.gaussian_matrix(n, n, seed))
    return q * np.sign(np.diag(r))[None, :]


def with_spectrum(sigma, seed_l, seed_r, m=None):
    n = len(sigma)
    m = m or n
    ql = orthogonal(m, seed_l)[:, :n]
    qr = orthogonal(n, seed_r)
    return (ql * np.asarray(sigma)[None, :]) @ qr.T


def sym_with_eigs(lam, seed):
    q = orthogonal(len(lam), seed)
    a = (q * np.asarray(lam)[None, :]) @ q.T
    return 0.5 * (a + a.T)


def geometric(n, kappa):
    return kappa ** (-np.arange(n) / (n - 1))


# ----------------------------------------------------------------- QDWH steps
def test_qr_step_matches_explicit_inverse_form():
    # test_polar.cpp:114-128: Eq. 2 (QR-based) == Eq. 1 X (aI + bX^TX)(I + cX^TX)^-1
    x = O.gaussian_matrix(30, 20, 11)
    x /= np.linalg.norm(x, 2)
    ell = 0.3
    w = qdwh.halley_weights(ell)
    g = x.T @ x
    ref = x @ (w.a * np.eye(20) + w.b * g) @ np.linalg.inv(np.eye(20) + w.c * g)
    got = qdwh.qdwh_qr_step(x, ell)
    assert np.linalg.norm(got - ref) <= 1e-11 * np.linalg.norm(ref)


def test_chol_step_matches_qr_step():
    # test_polar.cpp:130-135
    x = O.gaussian_matrix(40, 25, 12)
    x /= np.linalg.norm(x, 2)
    for ell in (0.2, 0.6):
        yc = qdwh.qdwh_chol_step(x, ell)
        yq = qdwh.qdwh_qr_step(x, ell)
        assert np.linalg.norm(yc - yq) <= 1e-10 * np.linalg.norm(yq)


def test_chol_step_fails_over_and_qr_step_survives():
    # test_polar.cpp:137-157: c ~ 1e20 makes Z = I + c X^T X numerically singular
    # for a rank-one X; scan weights for a witness, the QR step must survive it
    threw = False
    for ell in (1e-15, 1.5e-15, 2e-15, 3e-15, 5e-15, 7e-15):
        for rows in (2, 3, 4, 5):
            x = np.ones((rows, 2))
            try:
                qdwh.qdwh_chol_step(x, ell)
            except qdwh.NotPositiveDefinite:
                threw = True
                assert np.all(np.isfinite(qdwh.qdwh_qr_step(x, ell)))
    assert threw


def test_fixed_iterations_propagate_cholesky_failure():
    # polar.cpp:206-207: a fixed-iteration run never falls back — NotPositiveDefinite
    # from a Cholesky step propagates (the library checks the pivot flag once, after
    # the last step: the same exception, no per-step host round trip)
    witnesses = 0
    for ell in (1e-15, 1.5e-15, 2e-15, 3e-15, 5e-15, 7e-15):
        for rows in (2, 3, 4, 5):
            x = np.ones((rows, 2))
            try:
                qdwh.qdwh_chol_step(x, ell)
                continue
            except qdwh.NotPositiveDefinite:
                witnesses += 1
            with pytest.raises(qdwh.NotPositiveDefinite):
                qdwh.run_fixed_iterations(x, ell, 2, "CholeskyOnly")
    assert witnesses > 0


# ----------------------------------------------------------------- polar
def test_polar_recognizes_spd_and_orthogonal():
    # test_polar.cpp:159-178
    a = sym_with_eigs([1.0, 1.5, 2.0, 3.0, 4.0], 31)
    p = qdwh.polar_decompose(a, qdwh.PolarConfig(ell0=0.25))
    assert p.converged
    assert np.linalg.norm(p.up - np.eye(5)) <= 1e-13 * 5
    assert np.linalg.norm(p.up @ p.h - a) <= 1e-13 * np.linalg.norm(a)
    q = orthogonal(8, 32)
    p = qdwh.polar_decompose(q, qdwh.PolarConfig(ell0=1.0))
    assert p.converged
    assert np.linalg.norm(p.up - q) <= 1e-13 * 8
    assert np.linalg.norm(p.h - np.eye(8)) <= 1e-13 * 8


def test_polar_budget_on_ill_conditioned_matrix():
    # test_polar.cpp:180-197: kappa = 1e12, n = 200
    n = 200
    a = with_spectrum(geometric(n, 1e12), 41, 42)
    p = qdwh.polar_decompose(a, qdwh.PolarConfig(ell0=1e-12))
    assert p.converged and p.iters_qr + p.iters_chol <= 6
    assert np.linalg.norm(p.up @ p.h - a) <= 1e-13 * np.linalg.norm(a)
    assert np.linalg.norm(p.up.T @ p.up - np.eye(n)) / np.sqrt(n) <= 1e-13
    assert np.array_equal(p.h, p.h.T)
    tr = p.ell_trace
    assert all(tr[i + 1] > tr[i] and tr[i + 1] <= 1 + 16 * U for i in range(len(tr) - 1))


def test_polar_extra_step_is_idempotent():
    # test_polar.cpp:261-270
    n = 24
    a = with_spectrum(geometric(n, 100.0), 71, 72)
    p = qdwh.polar_decompose(a, qdwh.PolarConfig(ell0=0.01))
    again = qdwh.qdwh_chol_step(p.up, 1.0)
    assert np.linalg.norm(again - p.up) <= 10 * n * U


# ----------------------------------------------------------------- fixed iterations
def test_fixed_iterations_composed_maps():
    # test_polar.cpp:209-231
    r = qdwh.run_fixed_iterations(np.diag([-1.0, 1.0]), 0.2, 3, "CholeskyOnly")
    assert abs(r.x[0, 0] + 1) <= 1e-13 and abs(r.x[1, 1] - 1) <= 1e-13 and r.iters_chol == 3
    assert abs(O.composed_rational(-0.2, 0.2, 3) + 1) <= 1e-13
    r = qdwh.run_fixed_iterations(np.diag([-0.2, 0.9]), 0.2, 3, "CholeskyOnly")
    assert abs(r.x[0, 0] + 1) <= 1e-13
    r = qdwh.run_fixed_iterations(np.eye(3), 1.0, 1, "CholeskyOnly")
    assert np.linalg.norm(r.x - np.eye(3)) <= 1e-14 and abs(r.ell - 1) <= 1e-15


def test_matrix_drivers_equal_composed_rational():
    # test_polar.cpp:233-248
    for s in range(20):
        ell0 = 0.05 + 0.9 * s / 19.0
        g = O.gaussian_matrix(6, 1, 600 + s)[:, 0]
        d = ell0 + (1 - ell0) * (np.abs(g) - np.floor(np.abs(g)))
        iters = 1 + s % 3
        r = qdwh.run_fixed_iterations(np.diag(d), ell0, iters, "CholeskyOnly")
        for i in range(6):
            assert abs(r.x[i, i] - O.composed_rational(d[i], ell0, iters)) <= 1e-12


# ----------------------------------------------------------------- partial EIG
def gen_sym_eig(n, k, seed):
    """k negative eigenvalues of magnitude ~k, n-k positive ones in (0, n): the
    shape of the reference's gen_sym_eig_test (matgen.cpp)."""
    mag = np.abs(O.gaussian_matrix(4 * n, 1, seed)[:, 0]) + 0.1
    lam = np.empty(n)
    lam[:k] = -k * mag[:k]
    pos = n - k * mag[k:]
    pos = pos[pos > 0][: n - k]
    lam[k:] = pos
    return sym_with_eigs(lam, seed + 7), np.sort(lam)


@pytest.mark.parametrize("n,k,iters,rtol", [(256, 26, 3, 1e-12), (96, 10, 2, 1e-11)])
def test_partial_eig_synthetic(n, k, iters, rtol):
    # test_partial.cpp:73-102
    a, lam = gen_sym_eig(n, k, 100 + n)
    r = qdwh.qdwh_partial_eig(a, qdwh.choose_shift(iters))
    assert r.count() == k and r.subspace_size >= k
    np.testing.assert_allclose(r.lambda_minus, lam[:k], rtol=rtol)
    assert np.all(np.diff(r.lambda_minus) >= 0) and np.all(r.lambda_minus < 0)
    v = r.v
    norm2 = np.abs(lam).max()
    assert np.linalg.norm(np.eye(k) - v.T @ v) <= 1e-13 * np.sqrt(n)
    assert np.linalg.norm(a @ v - v * r.lambda_minus[None, :]) <= 1e-12 * norm2 * np.sqrt(n)


@pytest.mark.parametrize("n", [128, 256, 512])
def test_partial_eig_acceptance_sizes(n):
    # acceptance.cpp:106-128: k = n/10
    k = n // 10
    a, lam = gen_sym_eig(n, k, 200 + n)
    r = qdwh.qdwh_partial_eig(a, qdwh.choose_shift(3))
    assert r.count() == k
    np.testing.assert_allclose(r.lambda_minus, lam[:k], rtol=1e-10)


# ----------------------------------------------------------------- partial SVD
def test_partial_svd_diagonal():
    # test_partial.cpp:104-121
    r = qdwh.qdwh_partial_svd(np.diag([1.0, 0.5, 0.05]), 0.1)
    assert r.count() == 2
    np.testing.assert_allclose(r.sigma1, [1.0, 0.5], rtol=1e-12)


@pytest.mark.parametrize("s", [1e-1, 1e-2, 1e-3, 1e-4])
def test_partial_svd_thresholds(s):
    # acceptance.cpp:130-151: s in {1e-1 .. 1e-4}; cut is strict sigma > s * alpha
    n = 256
    sig = geometric(n, 1e6)
    a = with_spectrum(sig, 7, 8)
    r = qdwh.qdwh_partial_svd(a, s)
    cut = s * r.alpha
    expect = sig[sig > cut]
    margin = np.min(np.abs(sig - cut)) / cut
    if margin > 1e-8:  # the count is only well-defined away from the cut
        assert r.count() == len(expect)
        np.testing.assert_allclose(r.sigma1, expect, rtol=1e-12)
    u, v = r.u1, r.v1
    k = r.count()
    assert np.linalg.norm(a @ v - u * r.sigma1[None, :]) <= 1e-12 * np.sqrt(n) * sig[0]
    assert np.linalg.norm(np.eye(k) - u.T @ u) <= 1e-12 * np.sqrt(n)
    assert np.linalg.norm(np.eye(k) - v.T @ v) <= 1e-12 * np.sqrt(n)
