cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist_native.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_new.log 2>&1; echo rc=$? >> gpurun_out/pytest_new.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo rc=$? >> gpurun_out/bench_cfg2.err
tail -25 gpurun_out/pytest_new.log; tail -3 gpurun_out/bench_cfg2.err; cat gpurun_out/bench_cfg2.json | head -c 3000
