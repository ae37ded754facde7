"""Pin the CPU oracle (oracle/qdwh_oracle.py + oracle/qdwh_oracle.c) against the
golden vectors produced by the reference itself (tests/golden/make_golden.py)
and, when oracle/_ref/libqdwhref.so is present, against the live reference.

CPU only.  Bit-exact for the integer/libm layer (generator, Halley weights),
1e-10 relative for the floating-point pipeline (north-star tolerance)."""
import numpy as np
import pytest

from conftest import golden
from oracle import qdwh_oracle as O
from oracle import ref as R

EPS = np.finfo(float).eps


def test_gaussian_bit_exact():
    g = golden("gaussian")
    assert np.array_equal(O.gaussian_matrix(17, 5, 0), g["g1"])
    assert np.array_equal(O.gaussian_matrix(3, 11, 42), g["g2"])
    assert np.array_equal(O.gaussian_matrix(64, 1, 0x6C616E637A), g["g3"])
    assert np.array_equal(O.gaussian_matrix(64, 1, 0x6E6F726D32), g["g4"])


def test_gaussian_pure_python_matches_c():
    # math.log/cos are glibc, like the reference (kernels.cpp:28-32)
    for i in range(50):
        assert O.normal_draw(42, i) == O.gaussian_range(42, i, 1)[0]


def test_halley_weights_bit_exact():
    g = golden("scalars")
    for ell, w, it in zip(g["ells"], g["weights"], g["iters"]):
        ws = O.halley_weights(float(ell))
        assert [ws.a, ws.b, ws.c, ws.ell_in, ws.ell_out] == list(w)
        assert O.iterations_to_converge(float(ell), 5 * EPS) == it


def test_halley_known_answers():
    # test_polar.cpp:37-56
    w = O.halley_weights(1.0)
    assert abs(w.a - 3) <= 4 * EPS and abs(w.b - 1) <= 4 * EPS and abs(w.c - 3) <= 4 * EPS
    w = O.halley_weights(0.2)
    assert abs(w.a - 7.594) < 7.594e-3 and abs(w.b - 10.87) < 10.87e-3
    assert abs(w.c - 17.46) < 17.46e-3 and abs(w.ell_out - 0.9454) < 0.9454e-3
    assert O.iterations_to_converge(1e-15, 5 * EPS) <= 6
    with pytest.raises(ValueError):
        O.halley_weights(0.0)
    with pytest.raises(ValueError):
        O.halley_weights(1.5)


def test_composed_rational_flattens():
    # test_polar.cpp:250-259
    for s, iters in ((0.2, 3), (0.875, 2)):
        xs = -1.0 + np.arange(0, 10001, 50) / 10000.0
        worst = max(abs(O.composed_rational((1 - s) * x - s, s, iters) + 1.0) for x in xs)
        assert worst <= 1e-12


def test_kernels_against_reference():
    g = golden("kernels")
    q, r = O.qr_factor(g["a"])
    assert np.abs(q - g["q"]).max() < 1e-13
    assert np.abs(np.triu(r) - g["r"]).max() < 1e-13
    ql, rl = O.householder_qr_loop(g["a"])
    assert np.abs(ql - g["q"]).max() < 1e-13
    w = O.cholesky(g["z"])
    assert np.abs(w - g["w"]).max() < 1e-13 * np.abs(g["w"]).max()
    assert abs(O.two_norm_estimate(g["a"]) - float(g["norm2"])) < 1e-12 * float(g["norm2"])
    assert abs(O.lanczos_min_bound(g["lanczos_a"]) - float(g["lanczos"])) < 1e-10


def test_steps_against_reference():
    g = golden("steps")
    assert np.abs(O.qdwh_chol_step(g["x"], O.halley_weights(0.5)) - g["chol"]).max() < 1e-13
    assert np.abs(O.qdwh_qr_step(g["x"], O.halley_weights(0.5)) - g["qr"]).max() < 1e-13
    assert np.abs(O.qdwh_chol_step(g["xt"], O.halley_weights(0.3)) - g["chol_t"]).max() < 1e-13
    assert np.abs(O.qdwh_qr_step(g["xt"], O.halley_weights(1e-4)) - g["qr_t"]).max() < 1e-12
    f = golden("fixed")
    r = O.run_fixed_iterations(f["x0"], 0.2, 3, "CholeskyOnly")
    assert np.abs(r.x - f["x"]).max() < 1e-12
    assert np.array_equal(np.array(r.ell_trace), f["ell_trace"])


@pytest.mark.parametrize("name", ["polar_illcond", "polar_tall"])
def test_polar_against_reference(name):
    g = golden(name)
    p = O.polar_decompose(g["a"], ell0=float(g["ell0"]))
    assert p.iters_qr == int(g["iters_qr"]) and p.iters_chol == int(g["iters_chol"])
    assert np.array_equal(np.array(p.ell_trace), g["ell_trace"])
    # Up is only determined to u*cond(A) (cond up to 1e12 here): compare what is
    # well conditioned — H, the backward error and orthogonality (test_polar.cpp:180-197)
    a = g["a"]
    assert np.abs(p.h - g["h"]).max() < 1e-11 * np.abs(g["h"]).max()
    assert np.linalg.norm(p.up @ p.h - a) <= 1e-13 * np.linalg.norm(a)
    n = a.shape[1]
    assert np.linalg.norm(p.up.T @ p.up - np.eye(n)) / np.sqrt(n) <= 1e-13


EIG_CASES = ["eig_diag", "eig_spd", "eig_gen256", "eig_gen96_two_step", "eig_gen128_randomized",
             "eig_cfg1_n256", "eig_cfg2_n384", "eig_cfg4_wishart_n512", "eig_cfg4_wishart_n1024"]
SVD_CASES = ["svd_diag", "svd_identity", "svd_gen256", "svd_gen128_qrfirst",
             "svd_gen128_randomized", "svd_cfg3_n256", "svd_cfg5_tall"]


@pytest.mark.parametrize("name", EIG_CASES)
def test_partial_eig_against_reference(name):
    g = golden(name)
    r = O.qdwh_partial_eig(g["a"], O.choose_shift(int(g["iters"])), bool(g["randomize"]),
                           float(g["tol"]), int(g["seed"]))
    assert r.count() == len(g["lam"])
    if r.count():
        np.testing.assert_allclose(r.lambda_minus, g["lam"], rtol=1e-10)
        # same invariant subspace as the reference's V (stored for n <= 512)
        if g["v"].size:
            assert np.linalg.norm(r.v @ (r.v.T @ g["v"]) - g["v"]) < 1e-10 * np.sqrt(len(g["lam"]))
    assert abs(r.mu - float(g["mu"])) <= 1e-10 * abs(float(g["mu"]))
    assert r.subspace_size == int(g["subspace_size"])
    assert r.rank_index == int(g["rank_index"])
    assert r.iters_chol == int(g["iters_chol"])


@pytest.mark.parametrize("name", SVD_CASES)
def test_partial_svd_against_reference(name):
    g = golden(name)
    r = O.qdwh_partial_svd(g["a"], float(g["s"]), float(g["tol"]), bool(g["randomize"]),
                           int(g["seed"]))
    assert r.count() == len(g["sigma"])
    np.testing.assert_allclose(r.sigma1, g["sigma"], rtol=1e-10)
    assert abs(r.alpha - float(g["alpha"])) <= 1e-12 * float(g["alpha"])
    assert r.subspace_size == int(g["subspace_size"])
    assert (r.iters_qr, r.iters_chol) == (int(g["iters_qr"]), int(g["iters_chol"]))


def test_planted_spectra_recovered_by_reference():
    # the BASELINE config families at reduced size: the reference's values match the
    # planted spectrum, so the planted spectrum is a valid truth for large-n GPU tests
    g = golden("eig_cfg1_n256")
    lam = np.sort(g["planted"])[::-1][: int(g["k_want"])]
    np.testing.assert_allclose(float(g["shift_c"]) - g["lam"], lam, rtol=1e-12, atol=1e-13)
    g = golden("svd_cfg5_tall")
    np.testing.assert_allclose(g["sigma"], np.sort(g["planted"])[::-1][: int(g["k_want"])],
                               rtol=1e-12)


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
def test_live_reference_matches_oracle_small():
    a, _ = R.gen_sym_eig_test(48, 6, 901)
    lam, _, d = R.partial_eig(a, 3)
    r = O.qdwh_partial_eig(a, O.choose_shift(3))
    np.testing.assert_allclose(r.lambda_minus, lam, rtol=1e-10)
    a, _ = R.gen_svd_test(40, 4001)
    s, _, _, d = R.partial_svd(a, 0.1)
    r = O.qdwh_partial_svd(a, 0.1)
    np.testing.assert_allclose(r.sigma1, s, rtol=1e-10)


def _same_subspaces(v, w, lam, tol):
    """Columns of v and w span the same eigenspaces: per group of equal values
    (a cluster is compared through its projector, single values up to sign)."""
    i = 0
    n = len(lam)
    while i < n:
        j = i + 1
        while j < n and abs(lam[j] - lam[i]) <= 1e-9 * max(1.0, abs(lam[i])):
            j += 1
        p = v[:, i:j] @ v[:, i:j].T
        q = w[:, i:j] @ w[:, i:j].T
        assert np.abs(p - q).max() <= tol, (i, j, np.abs(p - q).max())
        i = j


def test_oracle_eig_full_pinned():
    # fullsolve.cpp:22-80 restated vs the reference's own qdwh_eig_full (two split levels)
    g = golden("full_eig")
    lam, v, depth = O.qdwh_eig_full(g["a"], int(g["base"]))
    assert depth == int(g["depth"]) == 2
    np.testing.assert_allclose(lam, g["lam"], rtol=0, atol=1e-12 * np.abs(g["lam"]).max())
    _same_subspaces(v, g["v"], g["lam"], 1e-10)
    np.testing.assert_allclose(g["lam"], np.sort(g["planted"]), atol=1e-12 * 4)


def test_oracle_svd_full_pinned():
    g = golden("full_svd")
    u, s, v = O.qdwh_svd_full(g["a"], int(g["base"]))
    np.testing.assert_allclose(s, g["sigma"], rtol=1e-10, atol=1e-14)
    _same_subspaces(v, g["v"], g["sigma"], 1e-8)
    _same_subspaces(u, g["u"], g["sigma"], 1e-8)


def test_oracle_accuracy_report_pinned():
    # metrics.cpp:58-100 (Eq. 5-7), both residual pairings, with and without delta
    g = golden("metrics")
    rep = O.accuracy_report(g["a"], g["u"], g["sigma"], g["v"], g["delta"], False)
    np.testing.assert_allclose(rep, g["report"], rtol=1e-6)
    rep = O.accuracy_report(g["a_sq"], g["v_sq"], g["lam_sq"], g["v_sq"], None, True)
    assert np.isnan(rep[2]) and np.isnan(g["report_paper"][2])
    np.testing.assert_allclose(np.delete(rep, 2), np.delete(g["report_paper"], 2), rtol=1e-6)
