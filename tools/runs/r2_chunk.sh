mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/r_chunk_bench.log 2>&1
grep '^{' gpurun_out/r_chunk_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['e2e']))"
