mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_multiprocess.py tests/test_gpu_fuzz.py -q -x -m gpu -p no:cacheprovider > gpurun_out/shard_k4l_tests.txt 2>&1; echo "tests rc=$?"; tail -n 3 gpurun_out/shard_k4l_tests.txt
for c in cfg5 cfg5a; do timeout 900 python tools/shard_budget.py --config $c --world 8 > gpurun_out/r2i_shard_budget_$c.json 2> gpurun_out/shard_budget_$c.err; echo "$c rc=$?"; cut -c1-300 gpurun_out/r2i_shard_budget_$c.json; python - <<PY
import json
d=json.load(open('gpurun_out/r2i_shard_budget_$c.json'))
print({k:d[k] for k in ('one_gpu_ms','phase1_max_ms','phase2_max_ms','estimated_step_ms','estimated_speedup')})
PY
done
