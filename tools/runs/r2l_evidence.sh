mkdir -p gpurun_out
NK=11 bash tools/round_profiles.sh r2l
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2l_smoke.txt 2>&1; tail -1 gpurun_out/r2l_smoke.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2l_pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/r2l_pytest_gpu.txt
timeout 2400 python tools/config_sweep.py --oracle --steps 10 > gpurun_out/r2l_config_sweep.jsonl 2> gpurun_out/r2l_config_sweep.err; echo "sweep rc=$?"
python tools/show_bench.py gpurun_out/r2l_bench.log | head -8; tail -2 gpurun_out/r2l_bench_reference.log | cut -c1-200
PGRID_FUZZ_BLOCKS=40 timeout 1800 python -m pytest tests/test_gpu_fuzz.py -q -m gpu -p no:cacheprovider > gpurun_out/r2l_fuzz_campaign.txt 2>&1; echo rc=$? >> gpurun_out/r2l_fuzz_campaign.txt; tail -n 2 gpurun_out/r2l_fuzz_campaign.txt
