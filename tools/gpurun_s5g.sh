cd $GRAFT_REPO_ROOT
for xp in 0 1; do
rm -f gpurun_out/dag4096.trace
QDWHG_DAG_XP=$xp QDWHG_DAG_TRACE=gpurun_out/dag4096.trace timeout 120 python tools/timeline.py fast 4096 > /dev/null 2>&1
echo "xp=$xp"; python tools/dag_trace.py gpurun_out/dag4096.trace 2>&1 | grep -E "span|acc|update  nr=128|utilisation"
done
