cd $GRAFT_REPO_ROOT
timeout 600 ncu --nvtx --nvtx-include "solve/" --set full --clock-control none --import-source on -k regex:lanczos_kernel -c 1 -o gpurun_out/lanczos_cfg2 python tools/ncu_solve.py --config 2 > gpurun_out/ncu_lz.log 2>&1; echo rc=$?
