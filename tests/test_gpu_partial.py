"""GPU parity of the QDWHpartial drivers (libqdwhg.so through the C ABI)
against the reference's golden vectors and the oracle, plus the north-star
gates: values within 1e-10 relative, ||AV - V L||_F/||A||_F <= 1e-12 sqrt(n),
||I - V^T V||_F <= 1e-12 sqrt(n).  Marked gpu."""
import numpy as np
import pytest

from conftest import golden
from oracle import qdwh_oracle as O
from paper_2104_14186_b200 import matgen, qdwh

pytestmark = pytest.mark.gpu

EIG_CASES = ["eig_diag", "eig_spd", "eig_gen256", "eig_gen96_two_step", "eig_gen128_randomized",
             "eig_cfg1_n256", "eig_cfg2_n384", "eig_cfg4_wishart_n512", "eig_cfg4_wishart_n1024"]
SVD_CASES = ["svd_diag", "svd_identity", "svd_gen256", "svd_gen128_qrfirst",
             "svd_gen128_randomized", "svd_cfg3_n256", "svd_cfg5_tall"]


def north_star_eig(a, lam, v):
    n, k = v.shape
    if k == 0:
        return
    res = np.linalg.norm(a @ v - v * lam) / np.linalg.norm(a)
    orth = np.linalg.norm(np.eye(k) - v.T @ v)
    assert res <= 1e-12 * np.sqrt(n), res
    assert orth <= 1e-12 * np.sqrt(n), orth


def north_star_svd(a, u, s, v):
    n = a.shape[1]
    k = len(s)
    if k == 0:
        return
    res = np.linalg.norm(a @ v - u * s) / np.linalg.norm(a)
    assert res <= 1e-12 * np.sqrt(n), res
    assert np.linalg.norm(np.eye(k) - v.T @ v) <= 1e-12 * np.sqrt(n)
    assert np.linalg.norm(np.eye(k) - u.T @ u) <= 1e-12 * np.sqrt(n)


@pytest.mark.parametrize("name", EIG_CASES)
def test_partial_eig_golden(name):
    g = golden(name)
    r = qdwh.qdwh_partial_eig(g["a"], qdwh.choose_shift(int(g["iters"])), bool(g["randomize"]),
                              float(g["tol"]), int(g["seed"]))
    assert r.count() == len(g["lam"])
    assert r.iters_chol == int(g["iters_chol"]) and r.iters_qr == 0
    assert abs(r.mu - float(g["mu"])) <= 1e-10 * abs(float(g["mu"]))
    assert r.ell_trace == list(g["ell_trace"]) or r.mu >= 0
    if r.count():
        np.testing.assert_allclose(r.lambda_minus, g["lam"], rtol=1e-10)
        north_star_eig(g["a"], r.lambda_minus, np.asarray(r.v))
        assert np.all(r.lambda_minus < 0) and np.all(np.diff(r.lambda_minus) >= 0)
        assert r.subspace_size >= r.count()


@pytest.mark.parametrize("name", SVD_CASES)
def test_partial_svd_golden(name):
    g = golden(name)
    r = qdwh.qdwh_partial_svd(g["a"], float(g["s"]), float(g["tol"]), bool(g["randomize"]),
                              int(g["seed"]))
    assert r.count() == len(g["sigma"])
    assert (r.iters_qr, r.iters_chol) == (int(g["iters_qr"]), int(g["iters_chol"]))
    assert abs(r.alpha - float(g["alpha"])) <= 1e-12 * float(g["alpha"])
    np.testing.assert_allclose(r.sigma1, g["sigma"], rtol=1e-10)
    north_star_svd(g["a"], np.asarray(r.u1), r.sigma1, np.asarray(r.v1))
    assert np.all(r.sigma1 > r.threshold * r.alpha)


def test_partial_eig_edge_cases():
    # test_partial.cpp:51-71
    r = qdwh.qdwh_partial_eig(np.diag([-0.5, 1.0, 2.0, 3.0]), qdwh.choose_shift(3))
    assert r.count() == 1 and abs(r.lambda_minus[0] + 0.5) <= 0.5e-13
    assert abs(abs(r.v[0, 0]) - 1) <= 1e-10 and np.all(np.abs(r.v[1:, 0]) <= 1e-10)
    r = qdwh.qdwh_partial_eig(np.diag(np.arange(1.0, 17.0)), qdwh.choose_shift(3))
    assert r.empty() and r.mu >= 0
    ns = np.eye(6)
    ns[0, 5] = 1.0
    with pytest.raises(ValueError):
        qdwh.qdwh_partial_eig(ns, qdwh.choose_shift(3))
    bad = np.eye(4)
    bad[1, 1] = np.nan
    with pytest.raises(ValueError):
        qdwh.qdwh_partial_eig(bad, qdwh.choose_shift(3))


def test_partial_svd_edge_cases():
    # test_partial.cpp:104-147
    a = O.gaussian_matrix(4, 4, 5)
    with pytest.raises(ValueError):
        qdwh.qdwh_partial_svd(a, 0.0)
    with pytest.raises(ValueError):
        qdwh.qdwh_partial_svd(a, 1.0)
    with pytest.raises(ValueError):
        qdwh.qdwh_partial_svd(O.gaussian_matrix(3, 4, 5), 0.1)
    r = qdwh.qdwh_partial_svd(np.diag([1.0, 1e-9, 1e-9]), 0.5)
    assert r.count() == 1
    r = qdwh.qdwh_partial_svd(np.eye(6), 0.5)
    assert r.count() == 6 and r.no_savings


def test_count_soundness():
    # test_partial.cpp:149-171 (reduced trial count)
    for s in range(8):
        n, k = 24, 2 + s % 8
        a, _ = O_gen_sym(n, k, 3000 + s)
        r = qdwh.qdwh_partial_eig(a, qdwh.choose_shift(3))
        assert r.count() == int(np.sum(np.linalg.eigvalsh(a) < 0))


def O_gen_sym(n, k, seed):
    # planted symmetric matrix with k negative eigenvalues (matgen.cpp:32-58 pattern)
    g = O.gaussian_range(seed ^ 0x6D61676E, 0, n)
    d = np.where(np.arange(n) < k, -k * (np.abs(g) + 0.1), n - k * (np.abs(g) + 0.1))
    d = np.where(d == 0, 1.0, d)
    q, _ = np.linalg.qr(O.gaussian_matrix(n, n, seed ^ 0x71316C65))
    a = (q * d) @ q.T
    return 0.5 * (a + a.T), d


def test_scale_equivariance():
    # test_partial.cpp:173-187
    sig = np.array([1.0, 0.8, 0.5, 0.3, 0.02, 0.01, 0.005])
    ql, _ = np.linalg.qr(O.gaussian_matrix(7, 7, 91))
    qr, _ = np.linalg.qr(O.gaussian_matrix(7, 7, 92))
    a = (ql * sig) @ qr.T
    base = qdwh.qdwh_partial_svd(a, 0.1)
    for gamma in (3.0, 0.25, 117.0):
        r = qdwh.qdwh_partial_svd(gamma * a, 0.1)
        assert r.count() == base.count()
        np.testing.assert_allclose(r.sigma1, gamma * base.sigma1, rtol=1e-12)


def test_randomized_equals_plain():
    d = np.array([5.0 + i for i in range(17)] + [-1.0 - (i % 3) for i in range(17, 20)])
    d = d[np.argsort(-np.abs(d))]
    a = np.diag(d)
    p = qdwh.qdwh_partial_eig(a, qdwh.choose_shift(3), False)
    r = qdwh.qdwh_partial_eig(a, qdwh.choose_shift(3), True, 0.01, 7)
    assert p.count() == r.count() and r.randomized and not p.randomized
    np.testing.assert_allclose(p.lambda_minus, r.lambda_minus, rtol=1e-12)


@pytest.mark.parametrize("n,frac,family", [(1024, 0.10, "uniform"), (2048, 0.01, "logsigned")])
def test_config_family_eig_vs_oracle(n, frac, family):
    """cfg1 exactly (n=1024, largest 103) and a cfg2-family instance at n=2048."""
    lam = matgen.config_eigenvalues(family, n, 42)
    k = int(np.ceil(frac * n)) if family == "uniform" else int(frac * n)
    c = matgen.largest_k_shift(lam, k)
    q, _ = np.linalg.qr(O.gaussian_matrix(n, n, 42))
    a = (q * lam) @ q.T
    a = 0.5 * (a + a.T)
    r = qdwh.partial_eig_request(a, "largest", c, k)
    ref = O.qdwh_partial_eig(c * np.eye(n) - a, O.choose_shift(3))
    assert r.count() == k and ref.count() == k
    np.testing.assert_allclose(r.lambda_minus, c - ref.lambda_minus, rtol=1e-10)
    np.testing.assert_allclose(r.lambda_minus, np.sort(lam)[::-1][:k], rtol=1e-10, atol=1e-14)
    north_star_eig(a, r.lambda_minus, np.asarray(r.v))


def test_device_pointer_path_matches_host(cuda):
    import torch
    g = golden("eig_gen256")
    r_host = qdwh.qdwh_partial_eig(g["a"], qdwh.choose_shift(3))
    ad = torch.from_numpy(np.asfortranarray(g["a"])).to(cuda)
    r_dev = qdwh.qdwh_partial_eig(ad, qdwh.choose_shift(3))
    assert torch.is_tensor(r_dev.v) and r_dev.v.is_cuda
    # the panel QR reduces with FP64 atomics: run-to-run differences are at rounding level
    np.testing.assert_allclose(r_dev.lambda_minus, r_host.lambda_minus, rtol=1e-13)
    vd, vh = r_dev.v.cpu().numpy(), r_host.v
    assert np.linalg.norm(vd @ (vd.T @ vh) - vh) < 1e-12


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_soak_multistream_paths(cuda, seed):
    """Repeated device-resident solves at sizes that take every concurrent path
    (QR look-ahead on the side stream, the Cholesky-step overlap at n in
    [2048, 5120], programmatic dependent launches): planted spectra recovered
    to 1e-10 and the north-star gates, run after run."""
    import torch
    from paper_2104_14186_b200 import matgen
    n = 3072
    lam = matgen.config_eigenvalues("logsigned", n, seed)
    k = 31
    c = matgen.largest_k_shift(lam, k)
    q = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device=cuda,
                                    generator=torch.Generator(device=cuda).manual_seed(seed)))[0]
    lt = torch.from_numpy(lam).to(cuda)
    a = (q * lt[None, :]) @ q.T
    a = (0.5 * (a + a.T)).t().contiguous().t()
    want = np.sort(lam)[::-1][:k]
    for _ in range(2):
        r = qdwh.partial_eig_request(a, "largest", c, k)
        assert r.count() == k
        np.testing.assert_allclose(r.lambda_minus, want, rtol=1e-10, atol=1e-14)
        v = r.v
        lam_k = torch.from_numpy(np.asarray(r.lambda_minus)).to(cuda)
        resid = torch.linalg.norm(a @ v - v * lam_k[None, :]) / torch.linalg.norm(a)
        orth = torch.linalg.norm(torch.eye(k, dtype=torch.float64, device=cuda) - v.T @ v)
        assert float(resid) <= 1e-12 * np.sqrt(n) and float(orth) <= 1e-12 * np.sqrt(n)
    # tall SVD through the same machinery (look-ahead QR of the stacked / tall operands)
    m2, n2 = 4096, 2048
    sig = 1.0 / np.arange(1, n2 + 1)
    u = torch.linalg.qr(torch.randn(m2, n2, dtype=torch.float64, device=cuda,
                                    generator=torch.Generator(device=cuda).manual_seed(seed + 10)))[0]
    w = torch.linalg.qr(torch.randn(n2, n2, dtype=torch.float64, device=cuda,
                                    generator=torch.Generator(device=cuda).manual_seed(seed + 20)))[0]
    b = ((u * torch.from_numpy(sig).to(cuda)[None, :]) @ w.T).t().contiguous().t()
    kk = 200
    rs = qdwh.partial_svd_request(b, cut=float(np.sqrt(sig[kk - 1] * sig[kk])))
    assert rs.count() == kk
    np.testing.assert_allclose(rs.sigma1, sig[:kk], rtol=1e-10)


@pytest.mark.parametrize("n,k,family", [(2048, 20, "logsigned"), (4096, 41, "logsigned"),
                                        (1536, 60, "uniform"), (1024, 103, "uniform")])
def test_cholqr_subspace_matches_householder(n, k, family):
    """The small-subspace extraction (Cholesky QR of B, projected Gaussian block)
    against the reference's Householder QR path (QDWHG_SUBSPACE_HOUSEHOLDER, in a
    subprocess so the switch is read fresh): same deficiency index and subspace
    size, eigenvalues to 1e-12, north-star gates on both."""
    import os
    import subprocess
    import sys
    code = (
        "import json, sys\n"
        "import numpy as np\n"
        "from oracle import qdwh_oracle as O\n"
        "from paper_2104_14186_b200 import matgen, qdwh\n"
        f"n, k, fam = {n}, {k}, '{family}'\n"
        "lam = matgen.config_eigenvalues(fam, n, 7)\n"
        "q, _ = np.linalg.qr(O.gaussian_matrix(n, n, 7))\n"
        "a = (q * lam) @ q.T\n"
        "a = 0.5 * (a + a.T)\n"
        "c = matgen.largest_k_shift(lam, k)\n"
        "r = qdwh.partial_eig_request(a, 'largest', c, k)\n"
        "v = np.asarray(r.v)\n"
        "res = np.linalg.norm(a @ v - v * r.lambda_minus) / np.linalg.norm(a)\n"
        "orth = np.linalg.norm(np.eye(r.count()) - v.T @ v)\n"
        "print(json.dumps(dict(vals=list(r.lambda_minus), ell=r.subspace_size, ind=r.rank_index,\n"
        "                      path=r.subspace_path,\n"
        "                      res=res, orth=orth, want=list(np.sort(lam)[::-1][:k]))))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for hh in (False, True):
        env = dict(os.environ, PYTHONPATH=root)
        env.pop("QDWHG_SUBSPACE_HOUSEHOLDER", None)
        if hh:
            env["QDWHG_SUBSPACE_HOUSEHOLDER"] = "1"
        p = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                           text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        import json
        outs.append(json.loads(p.stdout.strip().splitlines()[-1]))
    chq, hh = outs
    assert chq["path"] == 1 and hh["path"] == 0  # each run took the path under test
    assert len(chq["vals"]) == len(hh["vals"]) == k
    assert chq["ind"] == hh["ind"] and chq["ell"] == hh["ell"]
    np.testing.assert_allclose(chq["vals"], hh["vals"], rtol=1e-12)
    np.testing.assert_allclose(chq["vals"], chq["want"], rtol=1e-10, atol=1e-14)
    for o in outs:
        assert o["res"] <= 1e-12 * np.sqrt(n) and o["orth"] <= 1e-12 * np.sqrt(n)
