mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider > gpurun_out/bucket_tests.txt 2>&1; echo "bucket rc=$?"; tail -n 4 gpurun_out/bucket_tests.txt
for it in 256 512; do
PGRID_LOCAL_ITEMS=$it timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bucket_sort -c 1 -o gpurun_out/bk_$it python tools/ktimes.py --builds 1 > gpurun_out/ncu_bk_$it.log 2>&1; echo "ncu $it rc=$?"
done
