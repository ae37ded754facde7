cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "gemm or fullsize or cholqr" 2>&1 | tail -2
for c in 1 2; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-profile > gpurun_out/s5i_bench_cfg${c}.json 2> gpurun_out/s5i.err
  python -c "import json; d=json.loads(open('gpurun_out/s5i_bench_cfg${c}.json').read().strip().splitlines()[-1]); r=d['result']; print('cfg',$c, round(d['ms_per_step'],3), r.get('oracle_match'), r['resid'], [round(x*1e3,3) for x in r['stage_seconds'][:6]])"
done
