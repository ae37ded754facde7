cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for sl in 0 10 20 40 80; do
  for n in 2048 4096 8192; do
    echo "slack $sl n $n: $(QDWHG_DAG_SLACK=$sl timeout 120 python tools/timeline.py fast $n 2>&1 | grep chol_dag_kernel)"
  done
done
