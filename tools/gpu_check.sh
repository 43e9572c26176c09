#!/bin/bash
# One gpurun round-trip: GPU tests (fast subset unless FULL=1), then a bench line.
mkdir -p gpurun_out
if [ "${FULL:-0}" = "1" ]; then SEL="gpu"; else SEL="gpu and not slow"; fi
PGRID_SYNC_DEBUG=${SYNC:-0} timeout 900 python -m pytest tests -q -x -m "$SEL" -k "${K:-}" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --e2e-steps 3 ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
