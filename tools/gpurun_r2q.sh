cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --nvtx --nvtx-include "solve/" --set full --clock-control none --import-source on -k regex:gemm_dmma_kernel -c 14 -o gpurun_out/r02_gemm_solve_cfg2 python tools/ncu_solve.py --config 2 > gpurun_out/ncu_gemm2.log 2>&1; echo ncu rc=$?
grep -v "^[0-9]*\. " gpurun_out/ncu_gemm2.log | tail -4
python tools/ncu_gemm_traffic.py gpurun_out/r02_gemm_solve_cfg2.ncu-rep gpurun_out/r02_gemm_traffic_cfg2.json
