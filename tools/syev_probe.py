"""Time sym_eig_dense (Rayleigh-Ritz solver) on device-resident matrices and
check it: python tools/syev_probe.py n1 n2 ..."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_14186_b200 import qdwh  # noqa: E402

h = qdwh.Handle(0)
h.set_stream(torch.cuda.current_stream().cuda_stream)
for n in [int(x) for x in sys.argv[1:]]:
    rng = np.random.default_rng(n)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.sort(rng.uniform(-1, 1, n))
    a = (q * lam) @ q.T
    a = 0.5 * (a + a.T)
    A = torch.tensor(a, device="cuda").t().contiguous().t()
    for _ in range(3):
        vals, V = qdwh.sym_eig_dense(A, handle=h)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 10
    for _ in range(reps):
        vals, V = qdwh.sym_eig_dense(A, handle=h)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    Vh = V.cpu().numpy()
    err = np.max(np.abs(vals - lam))
    res = np.linalg.norm(a @ Vh - Vh * vals) / np.linalg.norm(a)
    orth = np.linalg.norm(Vh.T @ Vh - np.eye(n))
    print(f"n={n:4d} jac_max={os.environ.get('QDWHG_JACOBI_MAX', 'default')} {dt*1e6:9.1f} us  "
          f"val err {err:.1e} resid {res:.1e} orth {orth:.1e}")
