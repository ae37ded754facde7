"""One QDWHpartial solve of a BASELINE config bracketed by cudaProfilerStart/Stop,
for `ncu --profile-from-start off` captures of the solve's own kernels (the input
generation and warm-up stay outside):
    ncu --nvtx --nvtx-include "solve/" --set full -k regex:gemm_dmma_kernel -c 12 \
        python tools/ncu_solve.py --config 2"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2104_14186_b200 import qdwh  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=2)
a = p.parse_args()
dev = torch.device("cuda:0")
h = qdwh.Handle(device=0)
h.set_stream(torch.cuda.current_stream().cuda_stream)
inp = bench.make_input(a.config, dev, h)
bench.solve(inp, h)  # warm-up (task lists, arena)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
torch.cuda.nvtx.range_push("solve")
res = bench.solve(inp, h)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
torch.cuda.cudart().cudaProfilerStop()
print("k", res.count(), "stages", [round(x * 1e3, 3) for x in res.stage_seconds])
