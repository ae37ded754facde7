cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(nproc; free -g; lscpu | head -20; nvidia-smi -L) > gpurun_out/box.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --ignore=tests/test_gpu_fullsize.py > gpurun_out/pytest1.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest1.log
timeout 3300 python tests/golden/make_fullsize.py --cfg 1 2 3 5 4 --ref 1 2 --out gpurun_out/fullsize > gpurun_out/fullsize.log 2>&1; echo fullsize_rc=$? >> gpurun_out/fullsize.log
tail -3 gpurun_out/pytest1.log; tail -12 gpurun_out/fullsize.log
