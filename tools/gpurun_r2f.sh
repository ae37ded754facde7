cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/timeline.py fast 4096 > gpurun_out/tl_fast4096_dag.txt 2>&1; echo rc=$? >> gpurun_out/tl_fast4096_dag.txt
timeout 120 python -c "
import torch,sys; sys.path.insert(0,'.')
from paper_2104_14186_b200 import qdwh
h=qdwh.Handle(0); h.set_stream(torch.cuda.current_stream().cuda_stream)
for n in (256, 384, 1024, 4096, 8192):
    G=qdwh.gaussian_matrix_device(n,n,3,handle=h)
    Z=(G.T@G/n+torch.eye(n,dtype=torch.float64,device='cuda')).t().contiguous().t()
    Wi=qdwh.cholesky_inverse_fast(Z,handle=h)
    L=torch.linalg.cholesky(Z); ref=torch.linalg.inv(L.T)
    print(n, float((Wi-ref).abs().max()/ref.abs().max()), float(torch.tril(Wi,-1).abs().max()), flush=True)
" > gpurun_out/dag_check.txt 2>&1; echo rc=$? >> gpurun_out/dag_check.txt
cat gpurun_out/dag_check.txt; tail -16 gpurun_out/tl_fast4096_dag.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_dag.log 2>&1; echo rc=$? >> gpurun_out/pytest_dag.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_dag.json 2> gpurun_out/bench_cfg2_dag.err
tail -5 gpurun_out/pytest_dag.log; head -c 900 gpurun_out/bench_cfg2_dag.json; tail -3 gpurun_out/bench_cfg2_dag.err
