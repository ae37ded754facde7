cd $GRAFT_REPO_ROOT
for n in 1024 2048 4096; do
for g in 1 2 3 4 6; do
  echo "n=$n group=$g: $(QDWHG_DAG_GROUP=$g timeout 120 python tools/timeline.py fast $n 2>&1 | grep -E 'chol_dag_kernel|span' | tr '\n' ' ')"
done; done
for p in 3 2; do
for c in 2 1; do
  QDWHG_SUBSPACE_PASSES=$p timeout 600 python bench.py --config $c --no-cpu-baseline --no-profile > gpurun_out/s5d_bench_cfg${c}_p$p.json 2> gpurun_out/s5d.err
  python -c "import json; d=json.loads(open('gpurun_out/s5d_bench_cfg${c}_p$p.json').read().strip().splitlines()[-1]); r=d['result']; print('passes',$p,'cfg',$c, round(d['ms_per_step'],3), r.get('oracle_match'), r.get('max_rel_err_vs_oracle'), r['resid'], r['orth'], r['stage_seconds'][:3])"
done; done
