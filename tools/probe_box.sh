#!/bin/bash
# One-shot probe of a GPU box: host cores, GPU, FP64 DMMA/DFMA peak, cuBLAS DGEMM.
mkdir -p gpurun_out
{
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
./tools/fp64_peak
python - <<'PY'
import torch, time
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device='cuda'); b = torch.randn(n, n, dtype=torch.float64, device='cuda')
    for _ in range(3): torch.matmul(a, b)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(f"cuBLAS DGEMM n={n}: {2*n**3/best/1e9:.2f} TFLOP/s ({best:.2f} ms)")
    e0.record()
    for _ in range(20): torch.matmul(a, b)
    e1.record(); torch.cuda.synchronize()
    print(f"cuBLAS DGEMM n={n} sustained x20: {20*2*n**3/e0.elapsed_time(e1)/1e9:.2f} TFLOP/s")
PY
} 2>&1 | tee gpurun_out/probe.txt
