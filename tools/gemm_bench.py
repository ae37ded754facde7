"""DMMA GEMM engine vs cuBLAS DGEMM (torch) at the QDWH shapes.
python tools/gemm_bench.py [--n 4096] [--reps 10]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_14186_b200 import qdwh  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=4096)
p.add_argument("--reps", type=int, default=10)
p.add_argument("--only", default="")
a = p.parse_args()
dev = torch.device("cuda:0")
h = qdwh.Handle(0)
h.set_stream(torch.cuda.current_stream().cuda_stream)
n = a.n


def colmajor(t):
    return t.t().contiguous().t()


def timeit(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(a.reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for (m, nn, k, ta, tb) in [(n, n, n, False, False), (n, n, n, True, False), (n, n, n, False, True),
                           (n, n, n // 8, False, False), (2 * n, n, n, False, False)]:
    tag = f"{m}x{nn}x{k} {'T' if ta else 'N'}{'T' if tb else 'N'}"
    if a.only and a.only not in tag:
        continue
    A = colmajor(torch.randn((k, m) if ta else (m, k), dtype=torch.float64, device=dev))
    B = colmajor(torch.randn((nn, k) if tb else (k, nn), dtype=torch.float64, device=dev))
    C = colmajor(torch.zeros((m, nn), dtype=torch.float64, device=dev))
    ms = timeit(lambda: qdwh.gemm(A, B, C, trans_a=ta, trans_b=tb, handle=h))
    ref = (A.T if ta else A) @ (B.T if tb else B)
    err = (C - ref).abs().max().item()
    ms_cublas = timeit(lambda: torch.matmul(A.T if ta else A, B.T if tb else B))
    fl = 2.0 * m * nn * k
    print(f"{tag:22s} ours {fl/ms/1e9:6.2f} TF ({ms:7.3f} ms)   cuBLAS {fl/ms_cublas/1e9:6.2f} TF   err {err:.1e}")
