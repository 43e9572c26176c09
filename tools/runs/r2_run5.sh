mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/r5_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r5_bench.log
timeout 900 python tools/shard_budget.py --config cfg5 --world 8 > gpurun_out/shard_budget_cfg5.json 2> gpurun_out/shard_budget.err
timeout 900 python tools/shard_budget.py --config cfg5a --world 8 > gpurun_out/shard_budget_cfg5a.json 2>> gpurun_out/shard_budget.err
timeout 1200 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
CHK_TIMEOUT=1500 bash tools/checked_tests.sh
tail -2 gpurun_out/r5_bench.log | cut -c1-3000; cat gpurun_out/shard_budget_cfg5*.json; tail -3 gpurun_out/pytest_gpu.log
