"""Run one cfg solve with live GEMM profiling and a per-launch log; summarize by shape class."""
import os, sys, collections, re
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
log = "gpurun_out/gemm_launches.log"
os.makedirs("gpurun_out", exist_ok=True)
if os.path.exists(log):
    os.remove(log)
os.environ["QDWHG_PROFILE_LOG"] = log
import torch, bench
from paper_2104_14186_b200 import qdwh
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dev = torch.device("cuda:0")
h = qdwh.Handle(0); h.set_stream(torch.cuda.current_stream().cuda_stream)
inp = bench.make_input(cfg, dev, h)
bench.solve(inp, h); torch.cuda.synchronize()
h.profile(True); h.kernel_stats()
if os.path.exists(log): os.remove(log)
res = bench.solve(inp, h)
st = h.kernel_stats()
print("gemm total", st)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for ln in open(log):
    m = re.match(r"BM=(\d+) AK=(\d) BK=(\d) M=(\d+) N=(\d+) K=(\d+) kmode=(\d) omode=(\d) splits=(\d+) grid=(\d+) ms=([\d.]+) gflop=([\d.]+)", ln)
    if not m: continue
    g = m.groups()
    key = f"BM={g[0]} M={g[3]} N={g[4]} K={g[5]} km={g[6]} om={g[7]} sp={g[8]} grid={g[9]}"
    a = agg[key]; a[0] += 1; a[1] += float(g[10]); a[2] += float(g[11])
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{v[1]:8.3f} ms {v[0]:5d}x  {v[2]/v[1]:6.2f} TF  {100*v[1]/tot:5.1f}%  {k}")
