"""Per-kernel device time of sym_eig_dense (QDWH D&C) on an n x n Wishart-like matrix."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_14186_b200 import qdwh
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
dev = torch.device("cuda:0")
h = qdwh.Handle(0); h.set_stream(torch.cuda.current_stream().cuda_stream)
G = qdwh.gaussian_matrix_device(n, n, 7, handle=h)
S = (G.T @ G / n).t().contiguous().t()
S = (0.5 * (S + S.T)).t().contiguous().t()
vals, V = qdwh.sym_eig_dense(S, handle=h); torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile
t0 = time.time()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    vals, V = qdwh.sym_eig_dense(S, handle=h); torch.cuda.synchronize()
wall = time.time() - t0
ref = torch.linalg.eigvalsh(S)
print(f"n={n} wall {wall:.3f}s  max|dlam| {float((torch.from_numpy(vals).to(dev)-ref).abs().max()):.2e} orth {float(torch.linalg.norm(V.T@V-torch.eye(n,dtype=V.dtype,device=dev))):.2e}")
tot = {}
for e in prof.events():
    if e.device_type.name == "CUDA":
        k = e.name.replace("(anonymous namespace)::", "").split("(")[0].replace("qdwhg::", "")[:80]
        t = tot.setdefault(k, [0, 0.0]); t[0] += 1; t[1] += e.device_time_total
allt = sum(v[1] for v in tot.values())
print(f"kernels total {allt/1e3:.1f} ms")
for k, v in sorted(tot.items(), key=lambda x: -x[1][1])[:16]:
    print(f"{v[1]/1e3:9.2f} ms {v[0]:6d}x {k}")
