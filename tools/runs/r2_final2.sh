# round-2 evidence at HEAD
mkdir -p gpurun_out
R=${R:-r2h}
bash tools/round_profiles.sh $R
python tools/ncu_kernels.py gpurun_out/${R}_full.ncu-rep > gpurun_out/${R}_ncu_full_cfg3.json 2>/dev/null
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${R}_smoke.log
timeout 900 python tools/shard_budget.py --config cfg5 --world 8 > gpurun_out/${R}_shard_budget_cfg5.json 2>/dev/null
timeout 900 python tools/shard_budget.py --config cfg5a --world 8 > gpurun_out/${R}_shard_budget_cfg5a.json 2>/dev/null
CHK_TIMEOUT=1500 bash tools/checked_tests.sh
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/${R}_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/${R}_pytest_gpu.log
tail -2 gpurun_out/${R}_bench.log | cut -c1-300; tail -2 gpurun_out/${R}_pytest_gpu.log; tail -3 gpurun_out/checked_pytest.log
