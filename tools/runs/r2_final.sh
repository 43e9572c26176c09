# round-2 evidence at HEAD: bench, reference arm, launch list, ncu full capture, smoke,
# and the sharded harness on config 5 at world 1 (strong-scaling code path on hardware)
mkdir -p gpurun_out
R=${R:-r2e}
bash tools/round_profiles.sh $R
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${R}_smoke.log
timeout 900 python bench.py --config cfg5 --sharded --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/${R}_sharded_cfg5.log 2>&1; echo "rc=$?" >> gpurun_out/${R}_sharded_cfg5.log
python tools/ncu_kernels.py gpurun_out/${R}_full.ncu-rep > gpurun_out/${R}_ncu_full_cfg3.json 2>/dev/null
tail -2 gpurun_out/${R}_bench.log | cut -c1-400; tail -2 gpurun_out/${R}_bench_reference.log | cut -c1-300; tail -2 gpurun_out/${R}_smoke.log; tail -3 gpurun_out/${R}_sharded_cfg5.log | cut -c1-600
