cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_partial.py tests/test_gpu_fullsize.py -x -q -k "cholqr or fullsize" > gpurun_out/pytest_sub.log 2>&1; echo rc=$? >> gpurun_out/pytest_sub.log; tail -5 gpurun_out/pytest_sub.log
for c in 1 2; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2_cfg$c.json 2> gpurun_out/bench_r2_cfg$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_r2_cfg$c.json').read().strip().splitlines()[-1])
print('cfg$c', round(d['ms_per_step'],2),'ms', round(d['value'],2), 'TF e2e', round(d['e2e']['value'],2), 'match', d['result'].get('oracle_match'), d['result'].get('stage_seconds'))
"
done
