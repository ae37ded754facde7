cd $GRAFT_REPO_ROOT
for b in 4 8 12 16 24 32; do
echo band $b
QDWHG_GEMM_BAND=$b timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_dmma_kernel python tools/gemm_traffic_probe.py 4096 2>&1 | grep -E "dram__|duration" | head -12
done
