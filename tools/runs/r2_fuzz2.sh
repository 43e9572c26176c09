mkdir -p gpurun_out
L=paper_2403_10647_b200/_lib
LIBS="$L/libpgrid_kf0.so $L/libpgrid.so $L/libpgrid_kf0.so $L/libpgrid.so" bash tools/ab_libs.sh
grep -v '^"parity\|^  ' gpurun_out/ab.log | grep "==\|radix_scatter\|value"
PGRID_FUZZ_BLOCKS=80 timeout 2400 python -m pytest tests/test_gpu_fuzz.py -q -m gpu -p no:cacheprovider > gpurun_out/r2_fuzz_campaign.txt 2>&1; echo rc=$? >> gpurun_out/r2_fuzz_campaign.txt
PGRID_FUZZ_BLOCKS=24 PGRID_LIB=$PWD/paper_2403_10647_b200/_lib/libpgrid_checked.so timeout 2400 python -m pytest tests/test_gpu_fuzz.py -q -m gpu -p no:cacheprovider > gpurun_out/r2_fuzz_campaign_checked.txt 2>&1; echo rc=$? >> gpurun_out/r2_fuzz_campaign_checked.txt
tail -3 gpurun_out/r2_fuzz_campaign.txt; tail -3 gpurun_out/r2_fuzz_campaign_checked.txt
