cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/dag4096.trace gpurun_out/dag8192.trace
QDWHG_DAG_TRACE=gpurun_out/dag4096.trace timeout 120 python tools/timeline.py fast 4096 > /dev/null 2>&1
QDWHG_DAG_TRACE=gpurun_out/dag8192.trace timeout 120 python tools/timeline.py fast 8192 > /dev/null 2>&1
python tools/dag_trace.py gpurun_out/dag4096.trace; python tools/dag_trace.py gpurun_out/dag8192.trace
