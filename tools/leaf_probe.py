"""Small driver for ncu captures of the latency-bound leaf kernels
(potrf_diag_kernel, geqr2_panel_kernel): one n x n Cholesky-inverse and one QR."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_14186_b200 import qdwh  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dev = torch.device("cuda:0")
h = qdwh.Handle(0)
h.set_stream(torch.cuda.current_stream().cuda_stream)
G = qdwh.gaussian_matrix_device(n, n, 3, handle=h)
Z = (G.T @ G / n + torch.eye(n, dtype=torch.float64, device=dev)).t().contiguous().t()
for _ in range(2):
    W, Wi = qdwh.cholesky_factor_inverse(Z, handle=h)
    Q, R = qdwh.qr_factor(G, handle=h)
torch.cuda.synchronize()
print("ok", float((W.T @ W - Z).abs().max()), float((Q @ R - G).abs().max()))
