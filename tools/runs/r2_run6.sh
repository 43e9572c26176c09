mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/r6_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r6_bench.log
timeout 900 python tools/shard_budget.py --config cfg5 --world 8 > gpurun_out/shard_budget_cfg5.json 2> gpurun_out/shard_budget.err
timeout 900 python tools/shard_budget.py --config cfg5a --world 8 > gpurun_out/shard_budget_cfg5a.json 2>> gpurun_out/shard_budget.err
tail -3 gpurun_out/pytest_gpu.log; python tools/show_bench.py gpurun_out/r6_bench.log 2>/dev/null | head -5; cat gpurun_out/shard_budget_cfg5*.json | cut -c1-300
