"""W^{-1} of the fast Cholesky-and-inverse vs torch (fp64) at several n."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2104_14186_b200 import qdwh  # noqa: E402
h = qdwh.Handle(0)
h.set_stream(torch.cuda.current_stream().cuda_stream)
sizes = [int(x) for x in sys.argv[1:]] or [256, 384, 1024, 4096, 8192]
for n in sizes:
    G = qdwh.gaussian_matrix_device(n, n, 3, handle=h)
    Z = (G.T @ G / n + torch.eye(n, dtype=torch.float64, device='cuda')).t().contiguous().t()
    Wi = qdwh.cholesky_inverse_fast(Z, handle=h)
    L = torch.linalg.cholesky(Z)
    ref = torch.linalg.inv(L.T)
    print(n, float((Wi - ref).abs().max() / ref.abs().max()), float(torch.tril(Wi, -1).abs().max()), flush=True)
