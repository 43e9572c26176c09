mkdir -p gpurun_out
L=paper_2403_10647_b200/_lib
LIBS="$L/libpgrid_k1old.so $L/libpgrid.so $L/libpgrid_k1old.so $L/libpgrid.so" bash tools/ab_libs.sh
grep -v '^"parity\|^  ' gpurun_out/ab.log | grep "==\|boxes_count\|total\|value"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_inverted.py tests/test_gpu_fuzz.py -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_k1.log 2>&1; tail -2 gpurun_out/pytest_k1.log
