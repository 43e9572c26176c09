mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2i_pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/r2i_pytest_gpu.txt
timeout 2400 python tools/config_sweep.py --oracle --steps 10 > gpurun_out/r2i_config_sweep.jsonl 2> gpurun_out/r2i_config_sweep.err; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/r2i_config_sweep.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d.get('config') or d.get('name'), d.get('builds_per_s') or d.get('value'), d.get('parity'))
PY
tail -3 gpurun_out/r2i_config_sweep.err
timeout 900 python bench.py > gpurun_out/r2i_bench.log 2>&1; echo "bench rc=$?"; python tools/show_bench.py gpurun_out/r2i_bench.log 2>/dev/null | head -3
