cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/dag_check.py 1024 4096 8192 12288 > gpurun_out/dag_check.txt 2>&1; cat gpurun_out/dag_check.txt
for n in 8192 16384; do
  echo "n $n dag: $(timeout 120 python tools/timeline.py fast $n 2>&1 | grep -E 'span')"
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_dag.log 2>&1; echo rc=$? >> gpurun_out/pytest_dag.log; tail -3 gpurun_out/pytest_dag.log
for c in 2 1 3 4 5; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2_cfg$c.json 2> gpurun_out/bench_r2_cfg$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_r2_cfg$c.json').read().strip().splitlines()[-1])
print('cfg$c', round(d['ms_per_step'],2),'ms', round(d['value'],2), 'TF e2e', round(d['e2e']['value'],2), 'match', d['result'].get('oracle_match'), d['result'].get('stage_seconds'))
"
done
