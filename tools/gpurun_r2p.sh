cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r02_bench_cfg2.json 2> gpurun_out/r02_bench_cfg2.err; echo rc=$? >> gpurun_out/r02_bench_cfg2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_reference_cfg2.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-profile > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
python tools/launch_summary.py gpurun_out/r02_launches_cfg2.csv 20 > gpurun_out/r02_launches_cfg2_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_dmma_kernel -s 30 -c 20 -o gpurun_out/r02_gemm_cfg2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-profile > gpurun_out/ncu_gemm.log 2>&1; echo ncu2 rc=$?
python tools/ncu_gemm_traffic.py gpurun_out/r02_gemm_cfg2.ncu-rep gpurun_out/r02_gemm_traffic_cfg2.json > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chol_dag_kernel -c 1 -o gpurun_out/r02_chol_dag_cfg2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-profile > gpurun_out/ncu_dag.log 2>&1; echo ncu3 rc=$?
tail -2 gpurun_out/r02_bench_cfg2.err; head -c 600 gpurun_out/r02_bench_cfg2.json; echo; cat gpurun_out/r02_launches_cfg2_summary.txt | head -24
