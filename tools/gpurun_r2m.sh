cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/dag4096.trace
QDWHG_DAG_TRACE=gpurun_out/dag4096.trace timeout 120 python tools/timeline.py fast 4096 > /dev/null 2>&1
python tools/dag_trace.py gpurun_out/dag4096.trace | grep -v "^leaf k="
nvidia-smi -q -d CLOCK,POWER | grep -E "Graphics|SM |Power Draw|Power Limit|Clocks Event|Reasons" | head -20
