"""Generate the committed golden vectors by running THE REFERENCE ITSELF.

Run here (where /root/reference exists and `make -C oracle` has built
oracle/_ref/libqdwhref.so from the untouched reference sources):

    python tests/golden/make_golden.py

Each case stores its input bytes and the reference's outputs in one .npz.
The cases restate the reference's own known-answer tests
(proj/tests/test_partial.cpp, test_polar.cpp, test_kernels.cpp,
acceptance.cpp) plus small instances of the five BASELINE config families.
Inputs come from the reference's own generators (gen_sym_eig_test,
gen_svd_test, gaussian_matrix + qr_factor) so they are reference bytes too.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref as R  # noqa: E402
from paper_2104_14186_b200 import matgen  # noqa: E402


def sym_with_eigs(lam, seed):
    q = R.qr_factor(R.gaussian_matrix(len(lam), len(lam), seed))[0]
    a = (q * lam) @ q.T
    return 0.5 * (a + a.T)


def with_spectrum(sig, seed_l, seed_r):
    n = len(sig)
    ql = R.qr_factor(R.gaussian_matrix(n, n, seed_l))[0]
    qr = R.qr_factor(R.gaussian_matrix(n, n, seed_r))[0]
    return (ql * sig) @ qr.T


def save(name, **kw):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **kw)
    print("wrote", name)


def eig_case(name, a, iters=3, randomize=False, tol=0.01, seed=0, keep_v=True, **extra):
    lam, v, d = R.partial_eig(a, iters, randomize, tol, seed)
    if not keep_v:
        v = np.zeros((0, 0))
    save(name, kind="eig", a=a, iters=iters, randomize=randomize, tol=tol, seed=seed,
         lam=lam, v=v, mu=d["mu_or_alpha"], rank_index=d["rank_index"],
         subspace_size=d["subspace_size"], iters_chol=d["iters_chol"],
         borderline=d["borderline"], no_savings=d["no_savings"],
         ell_trace=np.array(d["ell_trace"]), **extra)


def svd_case(name, a, s, randomize=False, tol=0.01, seed=0, **extra):
    sig, u, v, d = R.partial_svd(a, s, tol, randomize, seed)
    save(name, kind="svd", a=a, s=s, randomize=randomize, tol=tol, seed=seed, sigma=sig, u=u,
         v=v, alpha=d["mu_or_alpha"], rank_index=d["rank_index"],
         subspace_size=d["subspace_size"], iters_qr=d["iters_qr"], iters_chol=d["iters_chol"],
         no_savings=d["no_savings"], ell_trace=np.array(d["ell_trace"]), **extra)


def main():
    # ---- scalar layer: Halley weights + iteration counts (test_polar.cpp:37-92)
    ells = np.concatenate([[1.0, 0.2, 0.875, 0.5, 1e-15, 1.16e-3, 0.151],
                           1e-12 * np.power(1e12, np.arange(50) / 49.0)])
    ells = np.minimum(ells, 1.0)
    w = np.array([R.halley_weights(float(e)) for e in ells])
    its = np.array([R.iterations_to_converge(float(e), 5 * np.finfo(float).eps) for e in ells])
    save("scalars", ells=ells, weights=w, iters=its)
    # ---- Gaussian generator (kernels.cpp:441-447), several seeds/shapes
    save("gaussian", g1=R.gaussian_matrix(17, 5, 0), g2=R.gaussian_matrix(3, 11, 42),
         g3=R.gaussian_matrix(64, 1, 0x6C616E637A), g4=R.gaussian_matrix(64, 1, 0x6E6F726D32))
    # ---- kernels
    a = R.gaussian_matrix(40, 24, 11)
    q, r = R.qr_factor(a)
    z = a.T @ a + np.eye(24)
    save("kernels", a=a, q=q, r=r, z=z, w=R.cholesky(z),
         norm2=R.two_norm_estimate(a),
         lanczos=R.lanczos_min_bound(sym_with_eigs(np.linspace(-1.0, 2.0, 48), 5)),
         lanczos_a=sym_with_eigs(np.linspace(-1.0, 2.0, 48), 5))
    # ---- single QDWH steps (polar.cpp:53-128) and fixed iterations
    x = with_spectrum(np.geomspace(1.0, 0.5, 32), 21, 22) * 0.9
    save("steps", x=x, chol=R.qdwh_chol_step(x, 0.5), qr=R.qdwh_qr_step(x, 0.5),
         xt=R.gaussian_matrix(48, 20, 7) / 12.0,
         chol_t=R.qdwh_chol_step(R.gaussian_matrix(48, 20, 7) / 12.0, 0.3),
         qr_t=R.qdwh_qr_step(R.gaussian_matrix(48, 20, 7) / 12.0, 1e-4))
    x0 = sym_with_eigs(np.linspace(-1.0, 1.0, 40), 9)
    fx, fd = R.run_fixed_iterations(x0, 0.2, 3, "CholeskyOnly")
    save("fixed", x0=x0, x=fx, ell_trace=np.array(fd["ell_trace"]))
    # ---- polar (test_polar.cpp:159-197)
    a = with_spectrum(np.geomspace(1.0, 1e-12, 96), 41, 42)
    up, h, d = R.polar(a, 1e-12)
    save("polar_illcond", a=a, up=up, h=h, alpha=d["mu_or_alpha"], iters_qr=d["iters_qr"],
         iters_chol=d["iters_chol"], ell_trace=np.array(d["ell_trace"]), ell0=1e-12)
    a = R.gaussian_matrix(80, 48, 77)
    up, h, d = R.polar(a, 1e-3)
    save("polar_tall", a=a, up=up, h=h, alpha=d["mu_or_alpha"], iters_qr=d["iters_qr"],
         iters_chol=d["iters_chol"], ell_trace=np.array(d["ell_trace"]), ell0=1e-3)
    # ---- partial EIG (test_partial.cpp:51-102, acceptance.cpp:106-128)
    eig_case("eig_diag", np.diag([-0.5, 1.0, 2.0, 3.0]))
    eig_case("eig_spd", np.diag(np.arange(1.0, 17.0)))
    a, dd = R.gen_sym_eig_test(256, 26, 1)
    eig_case("eig_gen256", a, planted=dd)
    a, dd = R.gen_sym_eig_test(96, 10, 3)
    eig_case("eig_gen96_two_step", a, iters=2, planted=dd)
    a, dd = R.gen_sym_eig_test(128, 13, 228)
    eig_case("eig_gen128_randomized", a, randomize=True, seed=7, planted=dd)
    # cfg1 / cfg2 families at reduced n through the shift map B = c I - A
    for name, n, fam, frac in (("eig_cfg1_n256", 256, "uniform", 0.10),
                               ("eig_cfg2_n384", 384, "logsigned", 0.01)):
        lam = matgen.config_eigenvalues(fam, n, 42)
        k = max(1, int(round(frac * n)))
        c = matgen.largest_k_shift(lam, k)
        q = R.qr_factor(R.gaussian_matrix(n, n, 42))[0]
        a = (q * lam) @ q.T
        a = 0.5 * (a + a.T)
        b = c * np.eye(n) - a
        eig_case(name, b, planted=lam, shift_c=c, k_want=k, a_orig=a)
    # ---- partial SVD (test_partial.cpp:104-139, acceptance.cpp:130-151)
    svd_case("svd_diag", np.diag([1.0, 0.5, 0.05]), 0.1)
    svd_case("svd_identity", np.eye(6), 0.5)
    a, dd = R.gen_svd_test(256, 2)
    svd_case("svd_gen256", a, 0.01, planted=dd)
    a, dd = R.gen_svd_test(128, 7)
    svd_case("svd_gen128_qrfirst", a, 5e-4, planted=dd)
    svd_case("svd_gen128_randomized", a, 0.01, randomize=True, seed=3, planted=dd)
    # cfg3 family (log-spaced 1 -> 1e-16) and cfg5 family (1/i, tall) at reduced size
    n = 256
    sig = matgen.config_singular_values("log16", n)
    a = with_spectrum(sig, 42 ^ 0x71316C65, 42 ^ 0x71327269)
    svd_case("svd_cfg3_n256", a,
             matgen.cut_fraction_s(sig, int(round(0.05 * n)), R.two_norm_estimate(a)),
             planted=sig, k_want=int(round(0.05 * n)))
    m, n = 384, 128
    sig = matgen.config_singular_values("inv", n)
    gl = R.gaussian_matrix(m, n, 42 ^ 0x71316C65)
    ul = R.qr_factor(gl)[0][:, :n]
    vr = R.qr_factor(R.gaussian_matrix(n, n, 42 ^ 0x71327269))[0]
    a = (ul * sig) @ vr.T
    svd_case("svd_cfg5_tall", a,
             matgen.cut_fraction_s(sig, int(round(0.10 * n)), R.two_norm_estimate(a)),
             planted=sig, k_want=int(round(0.10 * n)))


def wishart_cases():
    """cfg4 family (A = G^T G / n - I, G ~ N(0,1) seed 42) at n = 512 and 1024:
    the cfg4 recipe (c = 0.8881 - 0.05, B = c I - A, then the largest 20% by
    count) run through the reference itself."""
    for n in (512, 1024):
        g = R.gaussian_matrix(n, n, 42)
        a = g.T @ g / n - np.eye(n)
        a = 0.5 * (a + a.T)
        c = matgen.CONFIGS[4]["shift"]
        k = int(round(0.20 * n))
        b = c * np.eye(n) - a
        # (inputs are incompressible Gaussian bytes: no copy of A, and the
        # reference's vectors only at n = 512; the tests apply the north-star
        # gates to our own vectors)
        eig_case(f"eig_cfg4_wishart_n{n}", b, shift_c=c, k_want=k, keep_v=(n <= 512))


def full_cases():
    """fullsolve.cpp (qdwh_eig_full / qdwh_svd_full) and metrics.cpp
    (accuracy_report) run through the reference itself: a 96 x 96 symmetric
    matrix with a spread spectrum and a cluster (two levels of spectral
    divide-and-conquer at base 32), a 72 x 48 SVD, and the Eq. 5-7 report of a
    perturbed partial decomposition in both pairings."""
    n = 96
    lam = np.concatenate([np.linspace(-3.0, -0.5, 40), np.full(16, 0.25), np.linspace(1.0, 4.0, 40)])
    a = sym_with_eigs(lam, 77)
    lam_r, v_r, depth = R.eig_full(a, 32)
    save("full_eig", a=a, base=32, planted=lam, lam=lam_r, v=v_r, depth=depth)
    sig = np.logspace(0, -6, 48)
    b = with_spectrum(np.concatenate([sig, np.zeros(0)]), 78, 79)[:, :48]
    b = np.vstack([b, 1e-3 * R.gaussian_matrix(24, 48, 80)])
    u_r, s_r, vv_r = R.svd_full(b, 32)
    save("full_svd", a=b, base=32, u=u_r, sigma=s_r, v=vv_r)
    # metrics: a k = 10 partial SVD of b from the reference's full SVD, perturbed
    k = 10
    pu = u_r[:, :k] + 1e-9 * R.gaussian_matrix(b.shape[0], k, 81)
    pv = vv_r[:, :k] + 1e-9 * R.gaussian_matrix(b.shape[1], k, 82)
    ps = s_r[:k] * (1 + 1e-10 * np.arange(k))
    rep = R.accuracy_report(b, pu, ps, pv, s_r[:k], False)
    sq = a  # square case for the paper pairing: the symmetric eigen report (U = V)
    ev = v_r[:, -k:] + 1e-9 * R.gaussian_matrix(n, k, 83)
    rep_p = R.accuracy_report(sq, ev, lam_r[-k:], ev, None, True)
    save("metrics", a=b, u=pu, sigma=ps, v=pv, delta=s_r[:k], report=rep, a_sq=sq, v_sq=ev,
         lam_sq=lam_r[-k:], report_paper=rep_p)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "wishart":
        wishart_cases()
    elif len(sys.argv) > 1 and sys.argv[1] == "full":
        full_cases()
    else:
        main()
        wishart_cases()
        full_cases()
