#!/bin/bash
# The GPU test suite against the bounds-checked build (libpgrid_checked.so, -DPGRID_CHECKED=1:
# PG_ASSERT traps on any out-of-range shared / global index in the hot kernels) -- our stand-in
# for compute-sanitizer memcheck, which this GPU pool does not allow. Build it first with
# `make -C paper_2403_10647_b200/csrc checked` (the .so travels with the repo snapshot).
mkdir -p gpurun_out
PGRID_LIB=$PWD/paper_2403_10647_b200/_lib/libpgrid_checked.so timeout ${CHK_TIMEOUT:-1500} \
  python -m pytest tests -q -m gpu -p no:cacheprovider ${CHK_ARGS:-} > gpurun_out/checked_pytest.log 2>&1
echo "checked rc=$?" >> gpurun_out/checked_pytest.log
PGRID_LIB=$PWD/paper_2403_10647_b200/_lib/libpgrid_checked.so timeout 900 python tools/sanitize_drive.py \
  > gpurun_out/checked_drive.log 2>&1
echo "drive rc=$?" >> gpurun_out/checked_drive.log
tail -n 3 gpurun_out/checked_pytest.log gpurun_out/checked_drive.log
