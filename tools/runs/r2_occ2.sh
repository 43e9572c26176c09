mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu.log
L=paper_2403_10647_b200/_lib
LIBS="$L/libpgrid.so $L/libpgrid_k2m3.so $L/libpgrid.so $L/libpgrid_k2m3.so" bash tools/ab_libs.sh
grep -v '^"parity\|^  ' gpurun_out/ab.log | grep "==\|pairs_emit\|radix_scatter\|cell_offsets\|total\|value"
