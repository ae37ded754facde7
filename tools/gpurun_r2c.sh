cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/box.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q -rs --durations=15 > gpurun_out/pytest_all.log 2>&1; echo rc=$? >> gpurun_out/pytest_all.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo rc=$? >> gpurun_out/bench_cfg2.err
for cfg in 2 4; do
  timeout 900 python bench.py --dist --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dist_cfg$cfg.json 2> gpurun_out/bench_dist_cfg$cfg.err; echo rc=$? >> gpurun_out/bench_dist_cfg$cfg.err
done
tail -30 gpurun_out/pytest_all.log; tail -3 gpurun_out/bench_cfg2.err; head -c 2500 gpurun_out/bench_cfg2.json; for cfg in 2 4; do tail -2 gpurun_out/bench_dist_cfg$cfg.err; head -c 1500 gpurun_out/bench_dist_cfg$cfg.json; echo; done
