"""Every alternative code path behind a QDWHG_* environment switch, exercised
(each switch is read once per process, so each case runs in a fresh
subprocess) on solves that reach the switched code:

  * EIG n=3072 (Cholesky-step overlap window, CholQR subspace) and the same
    with randomized detection (Householder QR with look-ahead, grid panels),
  * tall SVD 4096 x 2048 with sigma_i = 1/i (tall QR, Rayleigh-Ritz SVD),
  * dense symmetric EIG n=300 on a clustered spectrum (tridiagonal path, the
    QDWH spectral divide-and-conquer fullsolve.cpp:22-80 when forced).

Values within 1e-10 of the planted spectra and the north-star gates, as on the
default path."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SNIPPET = r"""
import json, numpy as np, torch
from oracle import qdwh_oracle as O
from paper_2104_14186_b200 import matgen, qdwh
dev = torch.device("cuda", 0)
out = {}
n, k = 3072, 31
lam = matgen.config_eigenvalues("logsigned", n, 3)
q = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device=dev,
                                generator=torch.Generator(device=dev).manual_seed(3)))[0]
a = (q * torch.from_numpy(lam).to(dev)[None, :]) @ q.T
a = (0.5 * (a + a.T)).t().contiguous().t()
c = matgen.largest_k_shift(lam, k)
want = np.sort(lam)[::-1][:k]
for rnd in (False, True):
    r = qdwh.partial_eig_request(a, "largest", c, k, use_randomization=rnd, seed=11)
    v = r.v
    lt = torch.from_numpy(np.asarray(r.lambda_minus)).to(dev)
    out["eig%d" % rnd] = dict(
        k=r.count(), err=float(np.max(np.abs(np.asarray(r.lambda_minus) - want) / np.abs(want))),
        res=float(torch.linalg.norm(a @ v - v * lt[None, :]) / torch.linalg.norm(a)),
        orth=float(torch.linalg.norm(torch.eye(k, dtype=torch.float64, device=dev) - v.T @ v)))
m2, n2, kk = 4096, 2048, 200
sig = 1.0 / np.arange(1, n2 + 1)
u = torch.linalg.qr(torch.randn(m2, n2, dtype=torch.float64, device=dev,
                                generator=torch.Generator(device=dev).manual_seed(4)))[0]
w = torch.linalg.qr(torch.randn(n2, n2, dtype=torch.float64, device=dev,
                                generator=torch.Generator(device=dev).manual_seed(5)))[0]
b = ((u * torch.from_numpy(sig).to(dev)[None, :]) @ w.T).t().contiguous().t()
rs = qdwh.partial_svd_request(b, cut=float(np.sqrt(sig[kk - 1] * sig[kk])))
st = torch.from_numpy(np.asarray(rs.sigma1)).to(dev)
out["svd"] = dict(k=rs.count(), err=float(np.max(np.abs(np.asarray(rs.sigma1) - sig[:kk]) / sig[:kk])),
                  res=float(torch.linalg.norm(b @ rs.v1 - rs.u1 * st[None, :]) / torch.linalg.norm(b)))
ns = 300
ls = np.repeat(np.linspace(-1.0, 1.0, ns // 4), 4)[:ns] + 1e-9 * np.arange(ns)
qs, _ = np.linalg.qr(O.gaussian_matrix(ns, ns, 77))
s = (qs * ls) @ qs.T
s = 0.5 * (s + s.T)
vals, vv = qdwh.sym_eig_dense(s)
out["syev"] = dict(err=float(np.max(np.abs(vals - np.sort(ls)))),
                   res=float(np.linalg.norm(s @ vv - vv * vals) / np.linalg.norm(s)),
                   orth=float(np.linalg.norm(vv.T @ vv - np.eye(ns))))
print(json.dumps(out))
"""

SWITCHES = [("QDWHG_CHOL_NO_LAUUM", "1"), ("QDWHG_CHOL_STABLE", "1"),
            # the recursive Cholesky-and-inverse with the Z22 side-stream overlap (n = 3072
            # runs the tile-DAG kernel by default), with and without the overlap; DAG
            # sub-trees of <= 8 tiles under the recursion
            ("QDWHG_CHOL_NO_DAG", "1"), ("QDWHG_CHOL_NO_DAG,QDWHG_CHOL_NO_OVERLAP", "1"),
            ("QDWHG_CHOL_DAG_TMAX", "8"), ("QDWHG_DAG_GROUP", "2"),
            # the classic factor-then-invert leaf instead of the fused, pipelined one
            ("QDWHG_LEAF_NO_FUSED", "1"), ("QDWHG_LEAF_NO_FUSED,QDWHG_CHOL_NO_DAG", "1"),
            ("QDWHG_GEMM_NO_BALANCE", "1"), ("QDWHG_JACOBI_MAX", "8"), ("QDWHG_NO_PDL", "1"),
            ("QDWHG_NO_PRIORITY", "1"), ("QDWHG_PANEL_CAP", "32"), ("QDWHG_PANEL_SMEM", "1"),
            ("QDWHG_POTRF_NB", "64"), ("QDWHG_QR_NBO", "128"), ("QDWHG_QR_NO_LOOKAHEAD", "1"),
            ("QDWHG_QR_SIDE_CAP", "128"), ("QDWHG_SMALL_THREADS", "256"), ("QDWHG_SUBSPACE_PASSES", "2"),
            ("QDWHG_SUBSPACE_HOUSEHOLDER", "1"), ("QDWHG_SYEV_DC", "1")]


@pytest.mark.parametrize("var,val", SWITCHES)
def test_switched_path(var, val):
    env = dict(os.environ, PYTHONPATH=ROOT, **{v: val for v in var.split(",")})
    p = subprocess.run([sys.executable, "-c", SNIPPET], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    out = json.loads(p.stdout.strip().splitlines()[-1])
    gate_eig, gate_svd = 1e-12 * 3072 ** 0.5, 1e-12 * 2048 ** 0.5
    for key in ("eig0", "eig1"):
        r = out[key]
        assert r["k"] == 31 and r["err"] <= 1e-10, (key, r)
        assert r["res"] <= gate_eig and r["orth"] <= gate_eig, (key, r)
    assert out["svd"]["k"] == 200 and out["svd"]["err"] <= 1e-10 and out["svd"]["res"] <= gate_svd, out["svd"]
    sy = out["syev"]
    assert sy["err"] <= 1e-12 and sy["res"] <= 1e-12 and sy["orth"] <= 1e-12 * 300 ** 0.5, sy
