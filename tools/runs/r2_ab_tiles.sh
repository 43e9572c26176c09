mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
LIBS="paper_2403_10647_b200/_lib/libpgrid.so paper_2403_10647_b200/_lib/libpgrid_t384.so paper_2403_10647_b200/_lib/libpgrid_t512.so paper_2403_10647_b200/_lib/libpgrid.so" bash tools/ab_libs.sh
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/ab.log
