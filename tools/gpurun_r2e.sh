cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
QDWHG_DEBUG=1 python tools/timeline.py fast 4096 v > gpurun_out/tl_fast4096_dbg.txt 2> gpurun_out/tl_fast4096_dbg.err
wc -l gpurun_out/tl_fast4096_dbg.err
