cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "chol or dag or kernels" 2>&1 | tail -3
for n in 1024 2048 3072 4096; do
  echo "n=$n: $(timeout 120 python tools/timeline.py fast $n 2>&1 | grep -E 'chol_dag_kernel' | tr '\n' ' ')"
done
for c in 2 1; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-profile > gpurun_out/s5e_bench_cfg${c}.json 2> gpurun_out/s5e.err
  python -c "import json; d=json.loads(open('gpurun_out/s5e_bench_cfg${c}.json').read().strip().splitlines()[-1]); r=d['result']; print('cfg',$c, round(d['ms_per_step'],3), r.get('oracle_match'), r['resid'], r['stage_seconds'][:3])"
done
