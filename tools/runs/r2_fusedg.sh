# fused last pass (k_radix_scatter_g) vs separate K4: tests first, then per-kernel times and bench A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_fg.log 2>&1; echo rc=$? >> gpurun_out/pytest_fg.log
tail -3 gpurun_out/pytest_fg.log
for v in 0 1; do echo "== PGRID_FUSED_G=$v"; PGRID_FUSED_G=$v PGRID_KTIMES=1 timeout 300 python tools/ktimes.py | grep -v host; done
ENVS="PGRID_FUSED_G=0;PGRID_FUSED_G=1;PGRID_FUSED_G=0;PGRID_FUSED_G=1" bash tools/sweep_env.sh
grep -A1 "==" gpurun_out/sweep.log | grep -v "^--"
