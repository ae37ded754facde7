"""Per-kernel device time of one QDWHpartial solve (CUPTI via torch.profiler).
Usage: python tools/profile_solve.py [--config 2] [--steps 1]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2104_14186_b200 import qdwh  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=2)
p.add_argument("--steps", type=int, default=1)
a = p.parse_args()
dev = torch.device("cuda:0")
h = qdwh.Handle(device=0)
h.set_stream(torch.cuda.current_stream().cuda_stream)
inp = bench.make_input(a.config, dev, h)
for _ in range(2):
    res = bench.solve(inp, h)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.steps):
        res = bench.solve(inp, h)
    torch.cuda.synchronize()
tot = {}
for e in prof.events():
    if e.device_type.name == "CUDA":
        k = e.name.replace("(anonymous namespace)::", "").split("(")[0].replace("qdwhg::", "")[:90]
        t = tot.setdefault(k, [0, 0.0])
        t[0] += 1
        t[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
allt = sum(v[1] for v in tot.values())
print(f"solve wall (stage sum) {sum(res.stage_seconds)*1e3:.2f} ms; kernels total {allt/1e3/a.steps:.2f} ms/solve")
print("stages ms:", [round(x * 1e3, 3) for x in res.stage_seconds])
for k, v in sorted(tot.items(), key=lambda x: -x[1][1])[:30]:
    print(f"{v[1]/1e3/a.steps:9.3f} ms  {v[0]/a.steps:7.1f} launches  {k}")
