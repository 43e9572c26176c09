mkdir -p gpurun_out
timeout 2400 python tools/config_sweep.py --steps 10 > gpurun_out/r2_config_sweep.jsonl 2> gpurun_out/r2_config_sweep.err; echo rc=$? >> gpurun_out/r2_config_sweep.err
cat gpurun_out/r2_config_sweep.jsonl | cut -c1-400; tail -3 gpurun_out/r2_config_sweep.err
