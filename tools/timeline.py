"""Kernel timeline (start offset, duration, gap) of one library call via the
CUDA profiler: python tools/timeline.py chol|qr|potrf [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2104_14186_b200 import qdwh  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "chol"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
dev = torch.device("cuda:0")
h = qdwh.Handle(0)
h.set_stream(torch.cuda.current_stream().cuda_stream)
G = qdwh.gaussian_matrix_device(n, n, 3, handle=h)
X = (G / (G.norm() ** 0.5)).t().contiguous().t()
Z = (G.T @ G / n + torch.eye(n, dtype=torch.float64, device=dev)).t().contiguous().t()


Xs = ((G + G.T) / (2 * torch.linalg.matrix_norm(G, 2))).t().contiguous().t()
Ysvd = None
if what == "svd":
    m2 = int(sys.argv[4]) if len(sys.argv) > 4 else 8 * n
    q1, _ = qdwh.qr_factor(qdwh.gaussian_matrix_device(m2, n, 5, handle=h), handle=h)
    q2, _ = qdwh.qr_factor(qdwh.gaussian_matrix_device(n, n, 6, handle=h), handle=h)
    sig = 1.0 / torch.arange(1, n + 1, dtype=torch.float64, device=dev)
    Ysvd = ((q1[:, :n] * sig[None, :]) @ q2.T).t().contiguous().t()


inp = None
if what == "solve":  # one cfg2 solve (bench input)
    import bench
    inp = bench.make_input(2, dev, h)


def call():
    if what == "solve":
        import bench
        return bench.solve(inp, h)
    if what == "svd":
        return qdwh.svd_dense(Ysvd, handle=h)
    if what == "chol":
        return qdwh.qdwh_chol_step(X, 0.5, handle=h)
    if what == "sym":  # one symmetric Cholesky-based step (the EIG path)
        return qdwh.run_fixed_iterations(Xs, 0.2, 1, handle=h)
    if what == "fast":  # the recursive Cholesky-and-inverse of the QDWH step
        return qdwh.cholesky_inverse_fast(Z, handle=h)
    if what == "qr":
        return qdwh.qr_factor(G, handle=h)
    return qdwh.cholesky_factor_inverse(Z, handle=h)


for _ in range(3):
    call()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    call()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = t0
tot_gap = 0.0
agg = {}
for e in ev:
    st, en = e.time_range.start, e.time_range.end
    gap = st - prev_end
    tot_gap += max(gap, 0)
    name = e.name.replace("(anonymous namespace)::", "").split("(")[0].replace("qdwhg::", "")[:60]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += en - st
    if len(sys.argv) > 3 and sys.argv[3] == "v":
        print(f"{(st - t0):9.1f} us  dur {en - st:8.1f}  gap {gap:6.1f}  {name}")
    prev_end = max(prev_end, en)
print(f"span {prev_end - t0:.1f} us, busy {sum(v[1] for v in agg.values()):.1f} us, gaps {tot_gap:.1f} us")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:15]:
    print(f"{v[1]:9.1f} us {v[0]:5d}x  {k}")
