mkdir -p gpurun_out
for it in 8 100000000; do
  PGRID_LOCAL_ITEMS=$it PGRID_FUZZ_BLOCKS=30 timeout 1500 python -m pytest tests/test_gpu_fuzz.py -q -m gpu -p no:cacheprovider > gpurun_out/r2k_fuzz_items$it.txt 2>&1; echo rc=$? >> gpurun_out/r2k_fuzz_items$it.txt
  echo "items $it"; tail -n 3 gpurun_out/r2k_fuzz_items$it.txt
done
