mkdir -p gpurun_out
: > gpurun_out/ab.log
L=paper_2403_10647_b200/_lib
for lib in libpgrid_prev.so libpgrid.so libpgrid_prev.so libpgrid.so; do
  echo "== $lib" >> gpurun_out/ab.log
  PGRID_LIB=$PWD/$L/$lib PGRID_KTIMES=1 timeout 300 python tools/ktimes.py >> gpurun_out/ab.log 2>&1
  PGRID_LIB=$PWD/$L/$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_one.log 2>&1
  python tools/show_bench.py gpurun_out/ab_one.log 2>/dev/null | head -1 >> gpurun_out/ab.log
done
grep "==\|bucket_sort\|pairs_emit\|value" gpurun_out/ab.log
timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider > gpurun_out/bk_tests.txt 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/bk_tests.txt
