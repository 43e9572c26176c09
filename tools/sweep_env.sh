#!/bin/bash
# bench under several env settings: ENVS="A=1 B=2;A=2" bash tools/sweep_env.sh
mkdir -p gpurun_out; : > gpurun_out/sweep.log
IFS=';' read -ra SETS <<< "$ENVS"
for s in "${SETS[@]}"; do
  echo "== $s" >> gpurun_out/sweep.log
  env $s timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS:-} > gpurun_out/sweep_one.log 2>&1
  python tools/show_bench.py gpurun_out/sweep_one.log >> gpurun_out/sweep.log 2>&1
done
