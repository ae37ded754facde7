"""One plain n^3 DMMA GEMM (C = A B, column-major) for an ncu DRAM-traffic
capture: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    -k regex:gemm_dmma_kernel python tools/gemm_traffic_probe.py 4096"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_14186_b200 import qdwh  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
h = qdwh.Handle(0)
h.set_stream(torch.cuda.current_stream().cuda_stream)
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g).t().contiguous().t()
b = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g).t().contiguous().t()
c = torch.empty(n, n, dtype=torch.float64, device="cuda").t()
c = c.t().contiguous().t() if not c.is_contiguous() else c
c = torch.empty((n, n), dtype=torch.float64, device="cuda").t().contiguous().t()
qdwh.gemm(a, b, c, handle=h)
torch.cuda.synchronize()
err = (c - a @ b).abs().max().item()
print("n", n, "max err", err)
