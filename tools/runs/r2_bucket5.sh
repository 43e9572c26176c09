mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bucket.py -x -q -m gpu -p no:cacheprovider > gpurun_out/bucket_tests.txt 2>&1; echo "bucket rc=$?"; tail -n 2 gpurun_out/bucket_tests.txt
: > gpurun_out/ab.log
L=paper_2403_10647_b200/_lib
for cfg in "libpgrid_prev.so PGRID_LOCAL=1" "libpgrid.so PGRID_LOCAL=1" "libpgrid_prev.so PGRID_LOCAL=1" "libpgrid.so PGRID_LOCAL=1"; do
  set -- $cfg
  echo "== $cfg" >> gpurun_out/ab.log
  env $2 PGRID_LIB=$PWD/$L/$1 PGRID_KTIMES=1 timeout 300 python tools/ktimes.py >> gpurun_out/ab.log 2>&1
  env $2 PGRID_LIB=$PWD/$L/$1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_one.log 2>&1
  python tools/show_bench.py gpurun_out/ab_one.log 2>/dev/null | head -1 >> gpurun_out/ab.log
  grep -o '"parity": "[^"]*"' gpurun_out/ab_one.log | head -1 >> gpurun_out/ab.log
done
grep "==\|bucket_sort\|radix_scatter\|value\|parity" gpurun_out/ab.log
echo skip ncu
