cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on -k regex:chol_dag_kernel -c 1 -o gpurun_out/dag4096 python tools/timeline.py fast 4096 > gpurun_out/ncu_dag.log 2>&1
tail -3 gpurun_out/ncu_dag.log
ncu -i gpurun_out/dag4096.ncu-rep --page details --csv > gpurun_out/dag4096_details.csv 2>&1
grep -E "Duration|DMMA|Issue Slots Busy|Warp Cycles Per Issued|L2 Hit|Memory Throughput|Registers|Achieved Occupancy|dram__bytes" gpurun_out/dag4096_details.csv | head -30
