"""Per-kernel device time of one distributed QDWHpartial solve at world size 1
(grid 1 x 1, NCCL): python tools/profile_dist.py [--config 2] [--nb 512]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2104_14186_b200 import qdwh  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=2)
p.add_argument("--nb", type=int, default=512)
a = p.parse_args()
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("gloo", rank=0, world_size=1)
dev = torch.device("cuda:0")
h = qdwh.Handle(device=0)
h.set_stream(torch.cuda.current_stream().cuda_stream)
D = qdwh.Dist(h, 1, 1, a.nb, 0, unique_id=qdwh.dist_unique_id())
c = bench.config_desc(a.config)
inp = bench.make_input(a.config, dev, h)
A = inp["A"]
m, n = A.shape
D.load(A)


def solve():
    if c["kind"] == "eig":
        return D.partial_eig_request(None, "largest", inp["c"], inp["k"], n=n)
    return D.partial_svd_request(None, cut=inp["cut"], k=inp["k"], shape=(m, n))


solve()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    res = solve()
    torch.cuda.synchronize()
tot = {}
for e in prof.events():
    if e.device_type.name == "CUDA":
        k = e.name.replace("(anonymous namespace)::", "").split("(")[0].replace("qdwhg::", "")[:80]
        t = tot.setdefault(k, [0, 0.0])
        t[0] += 1
        t[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
allt = sum(v[1] for v in tot.values())
print(f"k {res.count()} stages {[round(x * 1e3, 2) for x in res.stage_seconds]} kernels {allt / 1e3:.2f} ms")
for k, v in sorted(tot.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{v[1] / 1e3:9.3f} ms {v[0]:6d}x  {k}")
dist.destroy_process_group()
