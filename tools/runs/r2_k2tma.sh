mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_inverted.py tests/test_gpu_fuzz.py tests/test_gpu_big.py -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_k2.log 2>&1; echo rc=$? >> gpurun_out/pytest_k2.log; tail -2 gpurun_out/pytest_k2.log
L=paper_2403_10647_b200/_lib
LIBS="$L/libpgrid_k2old.so $L/libpgrid.so $L/libpgrid_k2old.so $L/libpgrid.so" bash tools/ab_libs.sh
grep -v '^"parity\|^  ' gpurun_out/ab.log | grep "==\|pairs_emit\|total\|value"
