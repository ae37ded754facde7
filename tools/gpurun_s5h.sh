# final-evidence run of a session: full GPU suite, every config's bench line, the
# reference arm, ncu launch list + DAG capture of the bench command
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02final; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > $O/r02_pytest_gpu_summary.txt; tail -2 $O/r02_pytest_gpu_summary.txt
for c in 2 1 3 4 5; do
  timeout 900 python bench.py --config $c > $O/r02_bench_cfg$c.json 2> $O/r02_bench_cfg$c.err
  python -c "import json; d=json.loads(open('$O/r02_bench_cfg$c.json').read().strip().splitlines()[-1]); print($c, round(d['ms_per_step'],3), round(d['value'],2), round(d['e2e']['value'],2), d['result'].get('oracle_match'), round(d['roofline']['per_launch_mean_tflops'],2), round(d['roofline'].get('second_kernel',{}).get('achieved',0),2), d['result']['stage_seconds'][:6])"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/r02_bench_reference_cfg2.json 2>&1
tail -c 300 $O/r02_bench_reference_cfg2.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/r02_launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-profile > $O/ncu_launch.log 2>&1; echo ncu1 rc=$?
python tools/launch_summary.py $O/r02_launches_cfg2.csv 20 > $O/r02_launches_cfg2_summary.txt 2>&1; head -12 $O/r02_launches_cfg2_summary.txt
timeout 900 ncu --nvtx --nvtx-include "solve/" --set full --clock-control none --import-source on -k regex:chol_dag_kernel -c 1 -o $O/r02_chol_dag_cfg2 python tools/ncu_solve.py --config 2 > $O/ncu_dag.log 2>&1; echo ncu2 rc=$?
