cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/timeline.py fast 4096 v > gpurun_out/tl_fast4096.txt 2>&1
python tools/timeline.py sym 4096 v > gpurun_out/tl_sym4096.txt 2>&1
python tools/timeline.py solve 4096 > gpurun_out/tl_solve.txt 2>&1
tail -18 gpurun_out/tl_fast4096.txt; tail -18 gpurun_out/tl_sym4096.txt; cat gpurun_out/tl_solve.txt | tail -18
