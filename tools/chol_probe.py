import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_14186_b200 import qdwh
dev = torch.device("cuda:0")
h = qdwh.Handle(0); h.set_stream(torch.cuda.current_stream().cuda_stream)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
G0 = qdwh.gaussian_matrix_device(n, n, 3, handle=h)
Q, _ = qdwh.qr_factor(G0, handle=h)
s = 1.0 / torch.arange(1, n + 1, dtype=torch.float64, device=dev)
for cm in (False, True):
    A = (Q * s[None, :])
    if cm:
        A = A.t().contiguous().t()
    G = A.T @ A
    G = (0.5 * (G + G.T)).t().contiguous().t()
    L = torch.linalg.cholesky(G)
    for rep in range(3):
        W, Wi = qdwh.cholesky_factor_inverse(G, handle=h)
        D = (W - L.T).abs()
        idx = int(D.argmax()); i, j = idx % n, idx // n  # column-major? use unravel
        i, j = divmod(idx, n)
        R = (W.T @ W - G).abs()
        print("cm", cm, "rep", rep, "max|W-L^T|", float(D.max()), "at", (i, j),
              "W", float(W[i, j]), "L^T", float(L.T[i, j]),
              "resid", float(R.max()), "diag tail W", W.diagonal()[-3:].tolist(),
              "L", L.diagonal()[-3:].tolist(), flush=True)
