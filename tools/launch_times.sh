#!/bin/bash
# per-kernel device times of one cfg build (cold-cache, serialised) -> gpurun_out/launches.csv
python tools/prof_build.py --builds 1 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_build.py --builds 1 > gpurun_out/ncu_launch.log 2>&1
