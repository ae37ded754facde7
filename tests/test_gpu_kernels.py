"""GPU parity of the building blocks (libqdwhg.so through the C ABI) against the
reference's golden vectors and the oracle.  Marked gpu."""
import numpy as np
import pytest

from conftest import golden
from oracle import qdwh_oracle as O
from paper_2104_14186_b200 import qdwh

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
@pytest.mark.parametrize("m,n,k", [(64, 64, 64), (300, 257, 129), (1024, 512, 2048), (17, 900, 33)])
def test_gemm_dmma(cuda, ta, tb, m, n, k):
    import torch
    g = torch.Generator(device="cpu").manual_seed(m * 7 + n * 3 + k)
    A = torch.randn((k, m) if ta else (m, k), generator=g, dtype=torch.float64).to(cuda)
    B = torch.randn((n, k) if tb else (k, n), generator=g, dtype=torch.float64).to(cuda)
    C0 = torch.randn((m, n), generator=g, dtype=torch.float64).to(cuda)
    C = C0.t().contiguous().t()  # column-major
    Ac = A.t().contiguous().t()
    Bc = B.t().contiguous().t()
    qdwh.gemm(Ac, Bc, C, alpha=1.5, beta=-0.5, trans_a=ta, trans_b=tb)
    ref = 1.5 * ((A.T if ta else A) @ (B.T if tb else B)) - 0.5 * C0
    err = (C - ref).abs().max().item()
    assert err <= 1e-13 * max(1.0, ref.abs().max().item()) * np.sqrt(k), err


@pytest.mark.parametrize("m,n,k,out", [(2048, 2048, 1024, "full"), (2304, 2304, 768, "lower_mirror"),
                                       (2432, 1920, 640, "full"), (1200, 1200, 2048, "lower")])
def test_gemm_wave_balanced_tail(cuda, m, n, k, out):
    """Shapes whose last 128-tile wave is partial: full waves + split-K tail with
    compact partials and the per-tile reduction (alpha, beta Cin, diag, lower/mirror)."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(m + n + k)
    A = torch.randn((k, m), generator=g, dtype=torch.float64).to(cuda)
    B = torch.randn((k, n), generator=g, dtype=torch.float64).to(cuda)
    C0 = torch.randn((m, n), generator=g, dtype=torch.float64).to(cuda)
    C = C0.t().contiguous().t()
    qdwh.gemm(A.t().contiguous().t(), B.t().contiguous().t(), C, alpha=0.75, beta=0.25, trans_a=True,
              out=out, diag_add=2.0 if out != "full" else 0.0)
    ref = 0.75 * (A.T @ B) + 0.25 * C0
    if out != "full":
        ref = ref + 2.0 * torch.eye(m, dtype=torch.float64, device=cuda)
        low = torch.tril(torch.ones(m, n, dtype=torch.bool, device=cuda))
        if out == "lower_mirror":
            ref = torch.where(low, ref, ref.T)
        else:
            ref = torch.where(low, ref, C0)
    err = (C - ref).abs().max().item()
    assert err <= 1e-13 * max(1.0, ref.abs().max().item()) * np.sqrt(k), err


def test_qr_factor_matches_reference():
    g = golden("kernels")
    q, r = qdwh.qr_factor(g["a"])
    assert np.abs(q - g["q"]).max() < 1e-13
    assert np.abs(r - g["r"]).max() < 1e-13 * np.abs(g["r"]).max()
    assert np.all(np.tril(r, -1) == 0.0)


@pytest.mark.parametrize("m,n", [(200, 130), (513, 512), (1000, 64), (70, 70), (2048, 1000), (5000, 100)])
def test_qr_factor_identities(m, n):
    a = O.gaussian_matrix(m, n, 7 + m + n)
    q, r = qdwh.qr_factor(a)
    md = max(m, n)
    assert np.linalg.norm(q.T @ q - np.eye(m)) <= 50 * md * O.EPS
    assert np.linalg.norm(q @ r - a) <= 50 * md * O.EPS * np.linalg.norm(a)
    qn, rn = np.linalg.qr(a, mode="complete")
    # same reflector convention as the reference / LAPACK: same diag(R) signs
    np.testing.assert_allclose(np.diag(r), np.diag(rn), rtol=1e-10, atol=1e-12)


def test_cholesky_matches_reference():
    g = golden("kernels")
    w = qdwh.cholesky(g["z"])
    assert np.abs(w - g["w"]).max() < 1e-13 * np.abs(g["w"]).max()


@pytest.mark.parametrize("n", [50, 200, 1000, 1300])
def test_cholesky_random_spd(n):
    x = O.gaussian_matrix(n + 10, n, 3 + n)
    z = x.T @ x / n + np.eye(n)
    w = qdwh.cholesky(z)
    assert np.all(np.tril(w, -1) == 0.0) and np.all(np.diag(w) > 0)
    assert np.linalg.norm(w.T @ w - z) <= 1e-13 * n * np.linalg.norm(z)


@pytest.mark.parametrize("n", [700, 2048])
def test_cholesky_ill_conditioned(n):
    """Gram of Q diag(1/i): kappa = n^2.  The stable right-looking POTRF must be
    backward stable (no explicit-inverse multiplies), like the reference's
    dot-product Cholesky (kernels.cpp:124-146)."""
    q, _ = np.linalg.qr(O.gaussian_matrix(n, n, 11 + n))
    a = q / np.arange(1, n + 1)[None, :]
    z = a.T @ a
    z = 0.5 * (z + z.T)
    w, winv = qdwh.cholesky_factor_inverse(z)
    assert np.all(np.tril(w, -1) == 0.0) and np.all(np.diag(w) > 0)
    assert np.linalg.norm(w.T @ w - z) <= 1e-14 * n * np.linalg.norm(z)
    l = np.linalg.cholesky(z)
    np.testing.assert_allclose(np.diag(w), np.diag(l), rtol=1e-8)


def test_cholesky_torch_stream_order(cuda):
    """Device operands produced by queued torch work (clone, zero fill) right
    before the call must be visible to the library (stream ordering)."""
    import torch
    n = 1024
    q, _ = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device=cuda,
                                       generator=torch.Generator(device=cuda).manual_seed(5)))
    a = q / torch.arange(1, n + 1, dtype=torch.float64, device=cuda)[None, :]
    z = (a.T @ a)
    z = (0.5 * (z + z.T)).t().contiguous().t()
    l = torch.linalg.cholesky(z)
    for _ in range(4):
        w, _wi = qdwh.cholesky_factor_inverse(z)
        d = (w - l.T).abs().max().item()
        scratch = (w - l.T) * 1e6  # garbage for the allocator to hand back next round
        assert d <= 1e-12, d
        del scratch


def test_cholesky_indefinite_raises():
    z = np.eye(8)
    z[5, 5] = -1.0
    with pytest.raises(qdwh.NotPositiveDefinite):
        qdwh.cholesky(z)


@pytest.mark.parametrize("n", [2, 5, 30, 96, 160])
def test_sym_eig_jacobi(n):
    a = O.gaussian_matrix(n, n, 100 + n)
    s = 0.5 * (a + a.T)
    vals, v = qdwh.sym_eig_dense(s)
    ref = np.linalg.eigvalsh(s)
    np.testing.assert_allclose(vals, ref, rtol=0, atol=1e-13 * np.abs(ref).max() * n)
    assert np.linalg.norm(s @ v - v * vals) <= 1e-13 * np.linalg.norm(s) * n
    assert np.linalg.norm(v.T @ v - np.eye(n)) <= 1e-13 * n


@pytest.mark.parametrize("n", [17, 49, 132, 160, 161])
@pytest.mark.parametrize("kind", ["spread", "clustered"])
def test_sym_eig_small_tridiagonal(n, kind):
    """One-CTA tridiagonalisation path (17..160) and the cooperative one just above,
    with well-separated and tightly clustered spectra (inverse iteration + Lowdin)."""
    if kind == "spread":
        lam = np.linspace(-1.0, 1.0, n)
    else:
        lam = np.repeat(np.linspace(-1.0, 1.0, (n + 3) // 4), 4)[:n] + 1e-9 * np.arange(n)
    q, _ = np.linalg.qr(O.gaussian_matrix(n, n, 7 + n))
    s = (q * lam) @ q.T
    s = 0.5 * (s + s.T)
    vals, v = qdwh.sym_eig_dense(s)
    np.testing.assert_allclose(vals, np.sort(lam), rtol=0, atol=1e-13 * n)
    assert np.linalg.norm(s @ v - v * vals) <= 1e-13 * np.linalg.norm(s) * n
    assert np.linalg.norm(v.T @ v - np.eye(n)) <= 1e-13 * n


@pytest.mark.parametrize("n", [300, 700])
def test_sym_eig_divide_and_conquer(n):
    lam = np.linspace(-1.0, 2.0, n) + 0.001 * np.sin(np.arange(n))
    q, _ = np.linalg.qr(O.gaussian_matrix(n, n, 5))
    s = (q * lam) @ q.T
    s = 0.5 * (s + s.T)
    vals, v = qdwh.sym_eig_dense(s)
    np.testing.assert_allclose(vals, np.sort(lam), rtol=0, atol=1e-12)
    assert np.linalg.norm(s @ v - v * vals) <= 1e-12 * np.linalg.norm(s) * np.sqrt(n)
    assert np.linalg.norm(v.T @ v - np.eye(n)) <= 1e-12 * np.sqrt(n)


def test_sym_eig_rejects_nonsymmetric():
    s = np.eye(4)
    s[0, 3] = 1.0
    with pytest.raises(ValueError):
        qdwh.sym_eig_dense(s)


@pytest.mark.parametrize("m,n", [(40, 30), (300, 200)])
def test_svd_dense(m, n):
    a = O.gaussian_matrix(m, n, 9)
    u, s, v = qdwh.svd_dense(a)
    ref = np.linalg.svd(a, compute_uv=False)
    np.testing.assert_allclose(s, ref, rtol=1e-12)
    assert np.linalg.norm(u * s @ v.T - a) <= 1e-13 * np.linalg.norm(a) * np.sqrt(n)


def test_norm_and_lanczos_match_reference():
    g = golden("kernels")
    assert abs(qdwh.two_norm_estimate(g["a"]) - float(g["norm2"])) <= 1e-12 * float(g["norm2"])
    assert abs(qdwh.lanczos_min_bound(g["lanczos_a"]) - float(g["lanczos"])) <= 1e-10


def test_norm_estimate_brackets():
    # test_kernels.cpp:210-244
    for s in range(10):
        a = O.gaussian_matrix(30 + s, 20, 700 + s)
        est = qdwh.two_norm_estimate(a)
        truth = np.linalg.norm(a, 2)
        assert 0.99 * truth <= est <= 1.10 * truth
    with pytest.raises(ValueError):
        qdwh.two_norm_estimate(np.zeros((3, 3)))


def test_lanczos_lower_bound():
    for s in range(10):
        d = np.diag(np.linspace(-1 - s, 4, 40))
        assert qdwh.lanczos_min_bound(d) <= -1 - s + 1e-12
    assert qdwh.lanczos_min_bound(np.diag(np.arange(1.0, 9.0))) >= 0.0
    ns = np.eye(5)
    ns[0, 1] = 1.0
    with pytest.raises(ValueError):
        qdwh.lanczos_min_bound(ns)


def test_qdwh_steps_match_reference():
    g = golden("steps")
    np.testing.assert_allclose(qdwh.qdwh_chol_step(g["x"], 0.5), g["chol"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(qdwh.qdwh_qr_step(g["x"], 0.5), g["qr"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(qdwh.qdwh_chol_step(g["xt"], 0.3), g["chol_t"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(qdwh.qdwh_qr_step(g["xt"], 1e-4), g["qr_t"], rtol=0, atol=1e-12)


def test_qdwh_steps_identity_and_diagonal():
    # test_polar.cpp:94-112
    i4 = np.eye(4)
    assert np.linalg.norm(qdwh.qdwh_chol_step(i4, 1.0) - i4) <= 1e-14
    assert np.linalg.norm(qdwh.qdwh_qr_step(i4, 1.0) - i4) <= 1e-14
    w = qdwh.halley_weights(0.3)
    d = np.array([0.3, 0.55, 0.8, 1.0])
    yc = qdwh.qdwh_chol_step(np.diag(d), 0.3)
    yq = qdwh.qdwh_qr_step(np.diag(d), 0.3)
    r = d * (w.a + w.b * d * d) / (1 + w.c * d * d)
    np.testing.assert_allclose(np.diag(yc), r, rtol=1e-12)
    np.testing.assert_allclose(np.diag(yq), r, rtol=1e-12)


def test_fixed_iterations_match_reference():
    f = golden("fixed")
    r = qdwh.run_fixed_iterations(f["x0"], 0.2, 3, "CholeskyOnly")
    np.testing.assert_allclose(r.x, f["x"], rtol=0, atol=1e-12)
    assert r.ell_trace == list(f["ell_trace"])
    assert np.array_equal(r.x, r.x.T)  # symmetric input stays exactly symmetric


@pytest.mark.parametrize("name", ["polar_illcond", "polar_tall"])
def test_polar_matches_reference(name):
    g = golden(name)
    p = qdwh.polar_decompose(g["a"], qdwh.PolarConfig(ell0=float(g["ell0"])))
    assert (p.iters_qr, p.iters_chol) == (int(g["iters_qr"]), int(g["iters_chol"]))
    a = g["a"]
    n = a.shape[1]
    assert np.abs(p.h - g["h"]).max() < 1e-11 * np.abs(g["h"]).max()
    assert np.linalg.norm(p.up @ p.h - a) <= 1e-13 * np.linalg.norm(a)
    assert np.linalg.norm(p.up.T @ p.up - np.eye(n)) / np.sqrt(n) <= 1e-13
    assert np.array_equal(p.h, p.h.T)


@pytest.mark.parametrize("m,n,cond", [(300, 200, 1e8), (256, 256, 1e4)])
def test_polar_estimated_ell0(m, n, cond):
    """estimate_ell0: a certified lower bound of sigma_min(A)/||A||_2
    from the R factor, fewer QDWH iterations than the 1e-15 default, same polar factor."""
    u, _ = np.linalg.qr(O.gaussian_matrix(m, n, 61))
    v, _ = np.linalg.qr(O.gaussian_matrix(n, n, 62))
    sig = np.logspace(0, -np.log10(cond), n)
    a = (u * sig) @ v.T
    p0 = qdwh.polar_decompose(a)
    pe = qdwh.polar_decompose(a, qdwh.PolarConfig(estimate_ell0=True))
    ell0 = pe.ell_trace[0] * 1.10  # the trace starts at ell0 / 1.10 (polar.cpp:137)
    assert 0.0 < ell0 <= sig[-1] / sig[0] * 1.0000001
    assert ell0 >= 0.1 * sig[-1] / sig[0]  # within the 2x power-iteration margin (+ alpha)
    assert pe.iters_qr + pe.iters_chol < p0.iters_qr + p0.iters_chol
    # H is well conditioned (perturbations ~ u ||A||); Up moves by ~ u kappa
    assert np.abs(pe.h - p0.h).max() < 1e-12
    assert np.abs(pe.up - p0.up).max() < 1e-14 * cond
    assert np.linalg.norm(pe.up @ pe.h - a) <= 1e-13 * np.linalg.norm(a)
    assert np.linalg.norm(pe.up.T @ pe.up - np.eye(n)) / np.sqrt(n) <= 1e-13


def test_polar_config_errors():
    a = O.gaussian_matrix(4, 4, 51)
    with pytest.raises(ValueError):
        qdwh.polar_decompose(a, qdwh.PolarConfig(ell0=0.0))
    with pytest.raises(qdwh.NotConverged):
        qdwh.polar_decompose(a, qdwh.PolarConfig(ell0=1e-6, max_iters=1))
    with pytest.raises(ValueError):
        qdwh.polar_decompose(O.gaussian_matrix(3, 4, 1))


@pytest.mark.parametrize("nbo", ["128", "512"])
def test_qr_outer_block_sizes(nbo):
    """The 128/512-column outer blocking (512 is the default from n = 12288) on a
    small matrix, in a subprocess so the size knob is read fresh."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np\n"
        "from oracle import qdwh_oracle as O\n"
        "from paper_2104_14186_b200 import qdwh\n"
        "a = O.gaussian_matrix(1500, 1300, 91)\n"
        "q, r = qdwh.qr_factor(a)\n"
        "assert np.linalg.norm(q.T @ q - np.eye(1500)) <= 50 * 1500 * O.EPS\n"
        "assert np.linalg.norm(q @ r - a) <= 50 * 1500 * O.EPS * np.linalg.norm(a)\n"
        "qn, rn = np.linalg.qr(a, mode='complete')\n"
        "np.testing.assert_allclose(np.diag(r), np.diag(rn), rtol=1e-10, atol=1e-12)\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, QDWHG_QR_NBO=nbo, PYTHONPATH=root)
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_cholesky_inverse_fast_and_subspace_q2(cuda):
    """The two device building blocks of the distributed driver: the recursive
    Cholesky-and-inverse on a well-conditioned Z, and the partial.cpp:71-79 subspace
    extraction (ind, Q2) against the oracle's full QR."""
    import torch
    n = 700
    x = O.gaussian_matrix(n, n, 17) / np.sqrt(n)
    z = np.eye(n) + 3.0 * (x.T @ x)
    zi = qdwh.cholesky_inverse_fast(torch.from_numpy(np.asfortranarray(z)).to(cuda)).cpu().numpy()
    assert np.linalg.norm(zi.T @ z @ zi - np.eye(n)) <= 1e-12 * n
    assert np.allclose(np.tril(zi, -1), 0.0)
    # a rank-deficient "(X + I)/2"-like matrix: projector onto a 640-dim subspace
    q, _ = np.linalg.qr(O.gaussian_matrix(n, n, 18))
    lam = np.concatenate([np.ones(640), np.zeros(n - 640)])
    b = (q * lam) @ q.T
    ind, q2 = qdwh.subspace_q2(torch.from_numpy(np.asfortranarray(b)).to(cuda), 0.01)
    qo, ro = O.qr_factor(b)
    ind_o = O.detect_deficiency_index(ro, 0.01)
    assert ind == ind_o
    q2 = q2.cpu().numpy()
    ref = qo[:, ind - 1:]
    assert q2.shape == ref.shape
    assert np.linalg.norm(q2.T @ q2 - np.eye(q2.shape[1])) <= 1e-12 * n
    # same subspace: the projectors agree
    assert np.linalg.norm(q2 @ q2.T - ref @ ref.T) <= 1e-10


def test_device_gaussian_reference_stream_determinism_and_moments(cuda):
    """qdwhg_gaussian_matrix (kernels.cpp:441-447 counter scheme on the device;
    test_kernels.cpp:284-302 determinism and moments): the reference's own
    draws (golden, produced by the reference) to device-libm rounding, identical
    bits run to run, a different stream per seed, N(0,1) moments."""
    import torch
    g = golden("gaussian")
    for key, (m, n, seed) in {"g1": (17, 5, 0), "g2": (3, 11, 42), "g3": (64, 1, 0x6C616E637A),
                              "g4": (64, 1, 0x6E6F726D32)}.items():
        d = qdwh.gaussian_matrix_device(m, n, seed, device=cuda).cpu().numpy()
        np.testing.assert_allclose(d, g[key], rtol=1e-14, atol=1e-14)  # log/cospi vs glibc log/cos
    a = qdwh.gaussian_matrix_device(1500, 1000, 42, device=cuda)
    b = qdwh.gaussian_matrix_device(1500, 1000, 42, device=cuda)
    assert torch.equal(a, b)
    c = qdwh.gaussian_matrix_device(1500, 1000, 43, device=cuda)
    assert not torch.equal(a, c)
    np.testing.assert_allclose(a[:300, :200].cpu().numpy(), O.gaussian_matrix(1500, 1000, 42)[:300, :200],
                               rtol=1e-13, atol=1e-13)
    x = a.flatten().cpu().numpy()
    N = x.size
    assert abs(x.mean()) < 5.0 / np.sqrt(N)
    assert abs(x.var() - 1.0) < 5.0 * np.sqrt(2.0 / N)
    assert abs(np.mean(x ** 4) - 3.0) < 5.0 * np.sqrt(96.0 / N)
    assert abs(np.mean(x ** 3)) < 5.0 * np.sqrt(15.0 / N)


@pytest.mark.parametrize("n", [128, 200, 256, 384, 640, 1024, 3072, 4096, 4224, 8192])
def test_cholesky_inverse_fast_dag_sizes(cuda, n):
    """The tile-DAG Cholesky-and-inverse (chol_dag.cu) at every shape class: pure DAG
    launches (n = 128 T, T = 2 .. 32, K-step groups of 2 and 3), the recursion with a DAG
    sub-tree plus a non-DAG remainder (4224 = 4096 + 128), and two DAG sub-trees under
    the recursion (8192), a single fused leaf launch (128), a padded classic leaf under
    the recursion (200): W^{-1} against LAPACK on the kappa(Z) <= 1 + c class of the
    QDWH step (Z = I + c X^T X with c = 50)."""
    import torch
    x = torch.randn(n, n, dtype=torch.float64, device=cuda,
                    generator=torch.Generator(device=cuda).manual_seed(n))
    x = x / torch.linalg.matrix_norm(x, 2)
    z = (torch.eye(n, dtype=torch.float64, device=cuda) + 50.0 * (x.T @ x)).t().contiguous().t()
    wi = qdwh.cholesky_inverse_fast(z)
    ref = torch.linalg.inv(torch.linalg.cholesky(z).T)
    assert float((wi - ref).abs().max() / ref.abs().max()) <= 1e-13
    assert float(torch.tril(wi, -1).abs().max()) == 0.0
    r = wi.T @ z @ wi - torch.eye(n, dtype=torch.float64, device=cuda)
    assert float(torch.linalg.matrix_norm(r)) <= 1e-13 * n


@pytest.mark.parametrize("n", [128, 1024, 2176])
def test_cholesky_inverse_fast_repeatable(cuda, n):
    """The fused leaf runs its trailing updates and the rows of L^{-1} on warps that are
    only ordered by named barriers, and the DAG orders tiles by counters: any missing
    ordering would show as run-to-run differences.  30 launches on the same input must
    be bit-identical (single leaf launch, pure DAG, recursion + DAG + leaf)."""
    import torch
    x = torch.randn(n, n, dtype=torch.float64, device=cuda,
                    generator=torch.Generator(device=cuda).manual_seed(1000 + n))
    x = x / torch.linalg.matrix_norm(x, 2)
    z = (torch.eye(n, dtype=torch.float64, device=cuda) + 17.0 * (x.T @ x)).t().contiguous().t()
    first = qdwh.cholesky_inverse_fast(z).clone()
    for _ in range(30):
        again = qdwh.cholesky_inverse_fast(z)
        assert torch.equal(first, again)
