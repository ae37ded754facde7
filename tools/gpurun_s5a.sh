cd $GRAFT_REPO_ROOT
tools/bench_src/diag_bench | grep -A3 "fused"
rm -f gpurun_out/dag4096.trace gpurun_out/dag1024.trace
QDWHG_DAG_TRACE=gpurun_out/dag4096.trace timeout 120 python tools/timeline.py fast 4096 > /dev/null 2>&1
python tools/dag_trace.py gpurun_out/dag4096.trace | tail -22
QDWHG_DAG_TRACE=gpurun_out/dag1024.trace timeout 120 python tools/timeline.py fast 1024 > /dev/null 2>&1
python tools/dag_trace.py gpurun_out/dag1024.trace | tail -8
timeout 600 python -m pytest tests -m gpu -x -q -k "chol or dag or kernels" 2>&1 | tail -3
for c in 2 1; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/s5a_bench_cfg$c.json 2> gpurun_out/s5a_bench_cfg$c.err
  python -c "import json; d=json.loads(open('gpurun_out/s5a_bench_cfg$c.json').read().strip().splitlines()[-1]); print($c, round(d['ms_per_step'],3), round(d['value'],2), d['result'].get('oracle_match'), d['result']['stage_seconds'], round(d['roofline'].get('second_kernel',{}).get('achieved',0),2))"
done
