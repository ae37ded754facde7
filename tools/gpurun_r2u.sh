cd $GRAFT_REPO_ROOT
for g in 1 2 3 4 6; do
  echo "G=$g dag4096: $(QDWHG_DAG_KGROUP=$g timeout 120 python tools/timeline.py fast 4096 2>&1 | grep chol_dag_kernel) dag2048: $(QDWHG_DAG_KGROUP=$g timeout 120 python tools/timeline.py fast 2048 2>&1 | grep chol_dag_kernel)"
  QDWHG_DAG_KGROUP=$g python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --no-profile 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('  cfg2', d['ms_per_step'], d['result']['oracle_match'])"
done
