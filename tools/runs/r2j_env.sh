mkdir -p gpurun_out
: > gpurun_out/ab.log
for env in ${ENVS:-"PGRID_TC_PREF=0" "PGRID_TC_PREF=1" "PGRID_TC_PREF=0" "PGRID_TC_PREF=1"}; do
  echo "== $env" >> gpurun_out/ab.log
  env $env PGRID_KTIMES=1 timeout 300 python tools/ktimes.py >> gpurun_out/ab.log 2>&1
  env $env timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_one.log 2>&1
  python tools/show_bench.py gpurun_out/ab_one.log 2>/dev/null | head -1 >> gpurun_out/ab.log
  grep -o '"parity": "[^"]*"' gpurun_out/ab_one.log | head -1 >> gpurun_out/ab.log
done
grep "==\|tile_counts\|pairs_emit\|value\|parity" gpurun_out/ab.log
timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider > gpurun_out/bk_tests.txt 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/bk_tests.txt
