#!/bin/bash
# A/B of library variants: LIBS="a.so b.so" bash tools/ab_libs.sh -> gpurun_out/ab.log
: > gpurun_out/ab.log
for l in $LIBS; do
  echo "== $l" >> gpurun_out/ab.log
  PGRID_LIB=$l PGRID_KTIMES=1 timeout 300 python tools/ktimes.py ${KT_ARGS:-} >> gpurun_out/ab.log 2>&1
  PGRID_LIB=$l timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_one.log 2>&1
  python tools/show_bench.py gpurun_out/ab_one.log | head -1 >> gpurun_out/ab.log
  grep -o '"parity": "[^"]*"' gpurun_out/ab_one.log >> gpurun_out/ab.log
done
