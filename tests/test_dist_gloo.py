"""Multi-rank QDWHpartial (paper_2104_14186_b200/dist.py, 1D row blocks) at world
size 2 over gloo on CPU: same eigen/singular values as the single-process oracle
(1e-10 relative), north-star residual/orthogonality on the assembled vectors."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out_q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from dist_cpu_backend import CpuBackend
    from paper_2104_14186_b200 import dist as D
    comm = D.Comm(dist)
    be = CpuBackend()
    a = case["a"]
    m = a.shape[0]
    r0, r1 = D.row_range(m, rank, world)
    A_r = torch.from_numpy(np.ascontiguousarray(a[r0:r1]))
    if case["kind"] == "eig":
        res = D.dist_partial_eig(be, comm, A_r, m, s=0.2, iters=3)
        out = dict(values=res.values, v=None if res.v is None else res.v.numpy(),
                   ell=res.subspace_size, scale=res.scale)
    else:
        res = D.dist_partial_svd(be, comm, A_r, m, a.shape[1], s=case["s"])
        u = torch.zeros((m, len(res.values)), dtype=torch.float64)
        if res.u_rows is not None:
            u[r0:r1] = res.u_rows
        dist.all_reduce(u)
        out = dict(values=res.values, v=None if res.v is None else res.v.numpy(), u=u.numpy(),
                   ell=res.subspace_size, scale=res.scale)
    if rank == 0:
        out_q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def _run(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


def test_dist_partial_eig_matches_single_process():
    from oracle import qdwh_oracle as O
    from paper_2104_14186_b200 import matgen
    n = 96
    lam = matgen.config_eigenvalues("uniform", n, 42)
    q, _ = np.linalg.qr(O.gaussian_matrix(n, n, 42))
    a = (q * lam) @ q.T
    a = 0.5 * (a + a.T)
    k = 10
    c = matgen.largest_k_shift(lam, k)
    b = c * np.eye(n) - a
    out = _run(dict(kind="eig", a=b))
    ref = O.qdwh_partial_eig(b, O.choose_shift(3))
    assert len(out["values"]) == ref.count() == k
    np.testing.assert_allclose(out["values"], ref.lambda_minus, rtol=1e-10)
    v = out["v"]
    assert np.linalg.norm(b @ v - v * out["values"]) / np.linalg.norm(b) <= 1e-12 * np.sqrt(n)
    assert np.linalg.norm(v.T @ v - np.eye(k)) <= 1e-12 * np.sqrt(n)


def test_dist_partial_svd_tall_matches_single_process():
    from oracle import qdwh_oracle as O
    from paper_2104_14186_b200 import matgen
    m, n = 160, 64
    sig = matgen.config_singular_values("inv", n)
    ul, _ = np.linalg.qr(O.gaussian_matrix(m, n, 5))
    vr, _ = np.linalg.qr(O.gaussian_matrix(n, n, 6))
    a = (ul * sig) @ vr.T
    s = 0.05
    out = _run(dict(kind="svd", a=a, s=s))
    ref = O.qdwh_partial_svd(a, s)
    assert len(out["values"]) == ref.count()
    np.testing.assert_allclose(out["values"], ref.sigma1, rtol=1e-10)
    u, v, sv = out["u"], out["v"], out["values"]
    assert np.linalg.norm(a @ v - u * sv) / np.linalg.norm(a) <= 1e-12 * np.sqrt(n)
    assert np.linalg.norm(u.T @ u - np.eye(len(sv))) <= 1e-12 * np.sqrt(n)
    assert np.linalg.norm(v.T @ v - np.eye(len(sv))) <= 1e-12 * np.sqrt(n)


def test_row_partition():
    from paper_2104_14186_b200.dist import row_range
    for m in (1, 7, 64, 1001):
        for w in (1, 2, 3, 8):
            blocks = [row_range(m, r, w) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == m
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
