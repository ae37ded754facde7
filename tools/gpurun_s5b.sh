cd $GRAFT_REPO_ROOT
tools/bench_src/diag_bench | grep -A3 "potrf_diag_fused"
echo "=== qr 8192"; timeout 300 python tools/timeline.py qr 8192 2>&1 | tail -14
echo "=== cfg1"; timeout 300 python tools/profile_solve.py --config 1 2>&1 | tail -28
echo "=== cfg3"; timeout 300 python tools/profile_solve.py --config 3 2>&1 | tail -24
