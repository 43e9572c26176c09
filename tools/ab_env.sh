#!/bin/bash
# A/B of environment settings with per-kernel times: ENVS="A=1;A=0" bash tools/ab_env.sh -> gpurun_out/ab.log
: > gpurun_out/ab.log
IFS=';' read -ra SETS <<< "$ENVS"
for e in "${SETS[@]}"; do
  echo "== $e" >> gpurun_out/ab.log
  env $e PGRID_KTIMES=1 timeout 300 python tools/ktimes.py ${KT_ARGS:-} >> gpurun_out/ab.log 2>&1
  env $e timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ab_one.log 2>&1
  python tools/show_bench.py gpurun_out/ab_one.log | head -1 >> gpurun_out/ab.log
  grep -o '"parity": "[^"]*"' gpurun_out/ab_one.log >> gpurun_out/ab.log
done
