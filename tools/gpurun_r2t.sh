cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for c in 1 2 4; do
  python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print($c, d['ms_per_step'], d['result']['stage_seconds'], d['result']['oracle_match'], d['result'].get('max_rel_err_vs_oracle'))"
done
