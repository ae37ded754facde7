cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests -m gpu -x -q -k "dag_sizes" 2>&1 | tail -3
for n in 1024 2048 4096; do
  echo "n=$n: $(timeout 120 python tools/timeline.py fast $n 2>&1 | grep -E 'chol_dag_kernel' | tr '\n' ' ')"
done
rm -f gpurun_out/dag4096.trace
QDWHG_DAG_TRACE=gpurun_out/dag4096.trace timeout 120 python tools/timeline.py fast 4096 > /dev/null 2>&1
python tools/dag_trace.py gpurun_out/dag4096.trace > gpurun_out/dag4096.txt 2>&1; head -14 gpurun_out/dag4096.txt
for c in 2 1; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-profile > gpurun_out/s5f_bench_cfg${c}.json 2> gpurun_out/s5f.err
  python -c "import json; d=json.loads(open('gpurun_out/s5f_bench_cfg${c}.json').read().strip().splitlines()[-1]); r=d['result']; print('cfg',$c, round(d['ms_per_step'],3), r.get('oracle_match'), r['resid'], r['stage_seconds'][:3])"
done
