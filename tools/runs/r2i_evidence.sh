mkdir -p gpurun_out
NK=11 bash tools/round_profiles.sh r2i
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2i_smoke.txt 2>&1; tail -1 gpurun_out/r2i_smoke.txt
PGRID_LIB=$PWD/paper_2403_10647_b200/_lib/libpgrid_checked.so timeout 1800 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_parity.py tests/test_gpu_inverted.py tests/test_gpu_big.py -q -m gpu -p no:cacheprovider > gpurun_out/r2i_checked_build_pytest.txt 2>&1; echo "checked rc=$?"; tail -n 2 gpurun_out/r2i_checked_build_pytest.txt
python tools/show_bench.py gpurun_out/r2i_bench.log | head -8; tail -2 gpurun_out/r2i_bench_reference.log
