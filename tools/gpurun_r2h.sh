cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/dag_check.py > gpurun_out/dag_check.txt 2>&1; echo rc=$? >> gpurun_out/dag_check.txt
cat gpurun_out/dag_check.txt
rm -f gpurun_out/dag4096.trace gpurun_out/dag8192.trace
QDWHG_DAG_TRACE=gpurun_out/dag4096.trace timeout 120 python tools/timeline.py fast 4096 > /dev/null 2>&1
QDWHG_DAG_TRACE=gpurun_out/dag8192.trace timeout 120 python tools/timeline.py fast 8192 > /dev/null 2>&1
python tools/dag_trace.py gpurun_out/dag4096.trace; python tools/dag_trace.py gpurun_out/dag8192.trace
timeout 120 python tools/timeline.py fast 4096 2>&1 | tail -8
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_dag.json 2> gpurun_out/bench_cfg2_dag.err
head -c 700 gpurun_out/bench_cfg2_dag.json; grep -o '"stage_seconds[^]]*' gpurun_out/bench_cfg2_dag.json; tail -3 gpurun_out/bench_cfg2_dag.err
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_dag.log 2>&1; echo rc=$? >> gpurun_out/pytest_dag.log; tail -3 gpurun_out/pytest_dag.log
