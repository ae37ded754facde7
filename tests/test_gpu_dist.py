"""The multi-GPU driver's GPU backend (libqdwhg local ops + NCCL) at world size 1
on the single available B200: exercises every GpuBackend op on hardware; the
multi-rank orchestration itself is covered by tests/test_dist_gloo.py."""
import os
import socket

import numpy as np
import pytest

from oracle import qdwh_oracle as O
from paper_2104_14186_b200 import matgen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl1(cuda):
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    yield dist
    dist.destroy_process_group()


def test_dist_gpu_backend_eig(nccl1, cuda):
    import torch
    from paper_2104_14186_b200 import dist as D
    from paper_2104_14186_b200 import qdwh
    h = qdwh.Handle(0)
    h.set_stream(torch.cuda.current_stream().cuda_stream)
    be = D.GpuBackend(h)
    comm = D.Comm(nccl1)
    n, k = 512, 51
    lam = matgen.config_eigenvalues("uniform", n, 42)
    q, _ = np.linalg.qr(O.gaussian_matrix(n, n, 42))
    a = (q * lam) @ q.T
    a = 0.5 * (a + a.T)
    c = matgen.largest_k_shift(lam, k)
    b = c * np.eye(n) - a
    res = D.dist_partial_eig(be, comm, torch.from_numpy(b).to(cuda), n)
    ref = O.qdwh_partial_eig(b, O.choose_shift(3))
    assert len(res.values) == k
    np.testing.assert_allclose(res.values, ref.lambda_minus, rtol=1e-10)
    v = res.v.cpu().numpy()
    assert np.linalg.norm(b @ v - v * res.values) / np.linalg.norm(b) <= 1e-12 * np.sqrt(n)
    assert np.linalg.norm(v.T @ v - np.eye(k)) <= 1e-12 * np.sqrt(n)


def test_dist_gpu_backend_svd(nccl1, cuda):
    import torch
    from paper_2104_14186_b200 import dist as D
    from paper_2104_14186_b200 import qdwh
    h = qdwh.Handle(0)
    h.set_stream(torch.cuda.current_stream().cuda_stream)
    be = D.GpuBackend(h)
    comm = D.Comm(nccl1)
    m, n = 768, 256
    sig = matgen.config_singular_values("inv", n)
    ul, _ = np.linalg.qr(O.gaussian_matrix(m, n, 5))
    vr, _ = np.linalg.qr(O.gaussian_matrix(n, n, 6))
    a = (ul * sig) @ vr.T
    res = D.dist_partial_svd(be, comm, torch.from_numpy(a).to(cuda), m, n, s=0.02)
    ref = O.qdwh_partial_svd(a, 0.02)
    assert len(res.values) == ref.count()
    np.testing.assert_allclose(res.values, ref.sigma1, rtol=1e-10)
    u, v = res.u_rows.cpu().numpy(), res.v.cpu().numpy()
    assert np.linalg.norm(a @ v - u * res.values) / np.linalg.norm(a) <= 1e-12 * np.sqrt(n)
