"""Randomised parity sweep of the partial drivers through the C ABI: random sizes (40 .. 3000,
multiples of 128 and not), spectra (uniform, log-signed, clustered, gapped; harmonic, log,
deep-log = QR-first, gapped), fractions and the randomized-detection switch, against the
planted spectra: same k, values to 1e-12 ||A|| (EIG) / 1e-10 relative (SVD), the north-star
residual and orthogonality gates.  python tools/fuzz_partial.py SEED N_EIG N_SVD -> "FAILS n"."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2104_14186_b200 import qdwh
dev = torch.device("cuda:0")
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
fails = 0
def orth(n, seed):
    g = torch.randn(n, n, dtype=torch.float64, device=dev, generator=torch.Generator(device=dev).manual_seed(seed))
    return torch.linalg.qr(g)[0]
for trial in range(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    n = int(rng.choice([rng.integers(40, 300), rng.integers(300, 1200), rng.integers(1200, 3000), 128 * rng.integers(2, 20)]))
    kind = rng.choice(["uniform", "logsigned", "clustered", "gap"])
    frac = float(rng.choice([0.01, 0.05, 0.1, 0.2, 0.3]))
    k = max(1, int(round(frac * n)))
    if kind == "uniform":
        lam = rng.uniform(-1, 1, n)
    elif kind == "logsigned":
        lam = 10.0 ** rng.uniform(-8, 0, n) * rng.choice([-1.0, 1.0], n)
    elif kind == "clustered":
        lam = np.repeat(rng.uniform(-1, 1, (n + 3) // 4), 4)[:n] + 1e-7 * rng.standard_normal(n)
    else:
        lam = np.concatenate([rng.uniform(0.5, 1.0, k), rng.uniform(-1.0, 0.3, n - k)])
    lam_s = np.sort(lam)[::-1]
    if k >= n or lam_s[k - 1] - lam_s[k] < 1e-6 * max(1.0, abs(lam_s[k])):
        continue
    c = 0.5 * (lam_s[k - 1] + lam_s[k])
    q = orth(n, 1000 + trial)
    a = (q * torch.from_numpy(lam).to(dev)[None, :]) @ q.T
    a = (0.5 * (a + a.T)).t().contiguous().t()
    rnd = bool(rng.integers(0, 2))
    t0 = time.time()
    try:
        r = qdwh.partial_eig_request(a, "largest", float(c), k, use_randomization=rnd, seed=int(rng.integers(1, 1 << 30)))
        got = np.asarray(r.lambda_minus)
        ok = r.count() == k
        err = np.max(np.abs(got - lam_s[:k]) / np.maximum(np.abs(lam_s[:k]), 1e-300)) if ok else np.inf
        # relative to ||A||: tiny eigenvalues of the logsigned family cannot be relatively accurate beyond u ||A|| / |lambda|
        err_abs = np.max(np.abs(got - lam_s[:k])) / np.abs(lam).max() if ok else np.inf
        v = r.v
        lt = torch.from_numpy(got).to(dev)
        res = float(torch.linalg.norm(a @ v - v * lt[None, :]) / torch.linalg.norm(a)) / (1e-12 * np.sqrt(n)) if ok else np.inf
        orr = float(torch.linalg.norm(torch.eye(k, dtype=torch.float64, device=dev) - v.T @ v)) / (1e-12 * np.sqrt(n)) if ok else np.inf
        bad = (not ok) or err_abs > 1e-12 or res > 1 or orr > 1
        msg = f"k {r.count()}/{k} l {r.subspace_size} relerr {err:.1e} abserr {err_abs:.1e} res/gate {res:.3f} orth/gate {orr:.3f}"
    except Exception as e:  # noqa: BLE001
        bad = True
        msg = f"EXC {type(e).__name__}: {e}"
    fails += bad
    print(f"{'FAIL' if bad else 'ok  '} eig n={n} {kind} frac={frac} rnd={int(rnd)} {msg} ({time.time() - t0:.2f}s)", flush=True)
# SVD
for trial in range(int(sys.argv[3]) if len(sys.argv) > 3 else 25):
    n = int(rng.choice([rng.integers(40, 300), rng.integers(300, 1500), 128 * rng.integers(2, 12)]))
    m = int(n * rng.choice([1, 1, 2, 4])) + int(rng.integers(0, 5))
    kind = rng.choice(["harmonic", "log", "gap", "deep"])
    frac = float(rng.choice([0.02, 0.05, 0.1, 0.2]))
    if kind == "deep":
        frac = float(rng.choice([0.35, 0.4, 0.5]))
    k = max(1, int(round(frac * n)))
    if kind == "harmonic":
        sig = 1.0 / np.arange(1, n + 1)
    elif kind in ("log", "deep"):
        sig = 10.0 ** (-10.0 * np.arange(n) / (n - 1))
    else:
        sig = np.concatenate([np.sort(rng.uniform(0.5, 1.0, k))[::-1], np.sort(rng.uniform(0.0, 0.2, n - k))[::-1]])
    if sig[k - 1] / sig[k] < 1.0005:
        continue
    cut = float(np.sqrt(sig[k - 1] * sig[k]))
    if cut / sig[0] < 1.2e-3 and rng.integers(0, 2):
        pass
    gl = torch.randn(m, n, dtype=torch.float64, device=dev, generator=torch.Generator(device=dev).manual_seed(2000 + trial))
    u = torch.linalg.qr(gl)[0]
    w = orth(n, 3000 + trial)
    b = ((u * torch.from_numpy(sig).to(dev)[None, :]) @ w.T).t().contiguous().t()
    rnd = bool(rng.integers(0, 2))
    t0 = time.time()
    try:
        rs = qdwh.partial_svd_request(b, cut=cut, use_randomization=rnd, seed=int(rng.integers(1, 1 << 30)))
        got = np.asarray(rs.sigma1)
        ok = rs.count() == k
        err = np.max(np.abs(got - sig[:k]) / sig[:k]) if ok else np.inf
        st = torch.from_numpy(got).to(dev)
        res = float(torch.linalg.norm(b @ rs.v1 - rs.u1 * st[None, :]) / torch.linalg.norm(b)) / (1e-12 * np.sqrt(n)) if ok else np.inf
        ov = float(torch.linalg.norm(torch.eye(k, dtype=torch.float64, device=dev) - rs.v1.T @ rs.v1)) / (1e-12 * np.sqrt(n)) if ok else np.inf
        ou = float(torch.linalg.norm(torch.eye(k, dtype=torch.float64, device=dev) - rs.u1.T @ rs.u1)) / (1e-12 * np.sqrt(n)) if ok else np.inf
        bad = (not ok) or err > 1e-10 or res > 1 or ov > 1 or ou > 1
        msg = f"k {rs.count()}/{k} l {rs.subspace_size} relerr {err:.1e} res/gate {res:.3f} orthV {ov:.3f} orthU {ou:.3f} qr {rs.iters_qr} chol {rs.iters_chol}"
    except Exception as e:  # noqa: BLE001
        bad = True
        msg = f"EXC {type(e).__name__}: {e}"
    fails += bad
    print(f"{'FAIL' if bad else 'ok  '} svd {m}x{n} {kind} frac={frac} rnd={int(rnd)} {msg} ({time.time() - t0:.2f}s)", flush=True)
print("FAILS", fails)
