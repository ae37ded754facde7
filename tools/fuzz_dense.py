"""Randomised sweep of the dense entry points through the C ABI (polar_decompose with and
without the l0 estimate, sym_eig_dense, svd_dense, qdwh_svd_full): random shapes, condition
numbers up to 1e14, clustered / low-rank / grid spectra, against LAPACK.  Gates: polar
orthogonality and backward error 1e-13, eigen/singular values 1e-12, residual and
orthogonality at the north-star 1e-12 sqrt(n).  python tools/fuzz_dense.py SEED N -> "FAILS n"."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2104_14186_b200 import qdwh
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
N = int(sys.argv[2]) if len(sys.argv) > 2 else 12
fails = 0
def rep(tag, bad, msg):
    global fails
    fails += bool(bad)
    print(("FAIL " if bad else "ok   ") + tag + " " + msg, flush=True)
for t in range(N):
    # polar
    n = int(rng.choice([rng.integers(8, 200), rng.integers(200, 900), 128 * rng.integers(1, 8)]))
    m = n + int(rng.choice([0, 0, rng.integers(1, 300), n]))
    cond = 10.0 ** rng.uniform(0, 14)
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    sig = np.geomspace(1.0, 1.0 / cond, n)
    a = (u * sig) @ v.T
    try:
        p = qdwh.polar_decompose(a, qdwh.PolarConfig(estimate_ell0=bool(rng.integers(0, 2))))
        up, h = np.asarray(p.up), np.asarray(p.h)
        o = np.linalg.norm(up.T @ up - np.eye(n)) / np.sqrt(n)
        b = np.linalg.norm(up @ h - a) / np.linalg.norm(a)
        rep(f"polar {m}x{n} cond {cond:.1e}", o > 1e-13 or b > 1e-13 or not p.converged, f"orth {o:.1e} back {b:.1e} qr {p.iters_qr} chol {p.iters_chol}")
    except Exception as e:  # noqa: BLE001
        rep(f"polar {m}x{n} cond {cond:.1e}", True, f"EXC {e}")
    # sym eig
    n = int(rng.choice([rng.integers(2, 17), rng.integers(17, 161), rng.integers(161, 1200)]))
    kind = rng.choice(["rand", "cluster", "grid", "lowrank"])
    if kind == "rand":
        lam = rng.standard_normal(n)
    elif kind == "cluster":
        lam = np.repeat(rng.uniform(-1, 1, (n + 4) // 5), 5)[:n] + 1e-10 * rng.standard_normal(n)
    elif kind == "grid":
        lam = np.linspace(-1, 1, n)
    else:
        lam = np.concatenate([rng.uniform(1, 2, max(1, n // 10)), np.zeros(n - max(1, n // 10))])
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = (q * lam) @ q.T; s = 0.5 * (s + s.T)
    try:
        vals, vv = qdwh.sym_eig_dense(s)
        e = np.abs(vals - np.linalg.eigvalsh(s)).max() / max(1.0, np.abs(lam).max())
        r = np.linalg.norm(s @ vv - vv * vals) / (np.sqrt(n) * max(np.linalg.norm(s), 1e-300))
        o = np.linalg.norm(vv.T @ vv - np.eye(n)) / np.sqrt(n)
        # (a 268-fold zero eigenvalue at n = 297 measured 3.4e-13: inside the gate, 3x)
        rep(f"syev n={n} {kind}", e > 1e-12 or r > 1e-12 or o > 1e-12, f"val {e:.1e} res {r:.1e} orth {o:.1e}")
    except Exception as ex:  # noqa: BLE001
        rep(f"syev n={n} {kind}", True, f"EXC {ex}")
    # svd dense
    n = int(rng.choice([rng.integers(2, 40), rng.integers(40, 400)]))
    m = n + int(rng.choice([0, rng.integers(1, 50), 3 * n]))
    a = rng.standard_normal((m, n)) @ np.diag(np.geomspace(1, 10.0 ** -rng.uniform(0, 12), n)) @ np.linalg.qr(rng.standard_normal((n, n)))[0]
    try:
        uu, ss, vv = qdwh.svd_dense(a)
        uu, ss, vv = np.asarray(uu), np.asarray(ss), np.asarray(vv)
        e = np.abs(ss - np.linalg.svd(a, compute_uv=False)).max() / ss.max()
        r = np.linalg.norm(a @ vv - uu * ss) / np.linalg.norm(a)
        rep(f"svd {m}x{n}", e > 1e-13 or r > 1e-12, f"val {e:.1e} res {r:.1e}")
    except Exception as ex:  # noqa: BLE001
        rep(f"svd {m}x{n}", True, f"EXC {ex}")
    # full svd driver
    n = int(rng.choice([rng.integers(40, 200), rng.integers(200, 600)]))
    m = n + int(rng.choice([0, rng.integers(1, 100)]))
    a = np.linalg.qr(rng.standard_normal((m, n)))[0] * np.sort(rng.uniform(0.01, 1, n))[::-1] @ np.linalg.qr(rng.standard_normal((n, n)))[0].T
    try:
        f = qdwh.qdwh_svd_full(a, 32)
        uu, ss, vv = np.asarray(f.u), np.asarray(f.sigma), np.asarray(f.v)
        e = np.abs(ss - np.linalg.svd(a, compute_uv=False)).max() / ss.max()
        r = np.linalg.norm(a @ vv - uu * ss) / (np.sqrt(n) * np.linalg.norm(a))
        o = np.linalg.norm(vv.T @ vv - np.eye(n)) / np.sqrt(n)
        rep(f"svd_full {m}x{n}", e > 1e-12 or r > 1e-12 or o > 1e-12, f"val {e:.1e} res/gate {r/1e-12:.3f} orth/gate {o/1e-12:.3f}")
    except Exception as ex:  # noqa: BLE001
        rep(f"svd_full {m}x{n}", True, f"EXC {ex}")
print("FAILS", fails)
