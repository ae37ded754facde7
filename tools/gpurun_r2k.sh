cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/dag_check.py 1024 4096 > gpurun_out/dag_check.txt 2>&1; cat gpurun_out/dag_check.txt
for n in 2048 4096 8192; do
  echo "n $n dag: $(timeout 120 python tools/timeline.py fast $n 2>&1 | grep -E 'span')"
  echo "n $n rec: $(QDWHG_CHOL_NO_DAG=1 timeout 120 python tools/timeline.py fast $n 2>&1 | grep -E 'span')"
done
timeout 300 python tools/profile_solve.py --config 2 > gpurun_out/profile_cfg2.txt 2>&1; tail -32 gpurun_out/profile_cfg2.txt
