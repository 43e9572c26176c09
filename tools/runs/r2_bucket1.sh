mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bucket.py -x -q -m gpu -p no:cacheprovider > gpurun_out/bucket_tests.txt 2>&1; echo "bucket rc=$?"; tail -n 30 gpurun_out/bucket_tests.txt
: > gpurun_out/ab.log
for env in 0 1 0 1; do
  echo "== PGRID_LOCAL=$env" >> gpurun_out/ab.log
  PGRID_LOCAL=$env PGRID_KTIMES=1 timeout 300 python tools/ktimes.py >> gpurun_out/ab.log 2>&1
  PGRID_LOCAL=$env timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_one.log 2>&1
  python tools/show_bench.py gpurun_out/ab_one.log | head -1 >> gpurun_out/ab.log
  grep -o '"parity": "[^"]*"' gpurun_out/ab_one.log >> gpurun_out/ab.log
done
cat gpurun_out/ab.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_inverted.py tests/test_gpu_big.py -x -q -m gpu -p no:cacheprovider > gpurun_out/bucket_parity.txt 2>&1; echo "parity rc=$?"; tail -n 5 gpurun_out/bucket_parity.txt
