#!/bin/bash
# Evidence run for profiles/: bench line, reference arm, ncu launch list of the bench command,
# and one ncu --set full capture of every kernel of one cfg3 build. Usage: bash tools/round_profiles.sh r1
R=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/${R}_gpu.txt
timeout 900 python bench.py > gpurun_out/${R}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${R}_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${R}_bench_reference.log 2>&1; echo "ref rc=$?" >> gpurun_out/${R}_bench_reference.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/${R}_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/${R}_ncu_launch.log 2>&1
python tools/prof_build.py --builds 1 > gpurun_out/${R}_plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_" -s ${NK:-14} -c ${NK:-14} -o gpurun_out/${R}_full python tools/prof_build.py --builds 1 > gpurun_out/${R}_ncu_full.log 2>&1
echo done
