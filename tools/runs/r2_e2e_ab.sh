# A/B on one box: round-1 HEAD (tools/runs/r1, its own package + lib) vs this tree, bench lines
mkdir -p gpurun_out
for i in 1 2; do
  (cd tools/runs/r1 && timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 10) > gpurun_out/ab_r1_$i.log 2>&1
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/ab_r2_$i.log 2>&1
done
for f in gpurun_out/ab_r1_1.log gpurun_out/ab_r2_1.log gpurun_out/ab_r1_2.log gpurun_out/ab_r2_2.log; do
  echo "== $f"; python - "$f" <<'PY'
import json, sys
for ln in open(sys.argv[1]):
    if ln.startswith("{"):
        d = json.loads(ln); e = d["e2e"]
        print(d["value"], "builds/s", "e2e", e["value"], e.get("ms_per_step"), "seq", e.get("sequential_build_parallel_ms"),
              "pageable", e.get("pageable_build_parallel"))
PY
done
timeout 900 python tools/shard_budget.py --config cfg5 --world 8 > gpurun_out/shard_budget_cfg5.json 2> gpurun_out/shard_budget.err; tail -2 gpurun_out/shard_budget.err
cat gpurun_out/shard_budget_cfg5.json
timeout 1200 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
