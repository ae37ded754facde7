cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo rc=$? >> gpurun_out/pytest_all.log
for cfg in 2 4; do
  timeout 900 python bench.py --dist --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dist_cfg$cfg.json 2> gpurun_out/bench_dist_cfg$cfg.err; echo rc=$? >> gpurun_out/bench_dist_cfg$cfg.err
done
tail -5 gpurun_out/pytest_all.log; for cfg in 2 4; do tail -2 gpurun_out/bench_dist_cfg$cfg.err; head -c 1500 gpurun_out/bench_dist_cfg$cfg.json; echo; done
