mkdir -p gpurun_out
PGRID_FUZZ_BLOCKS=80 timeout 2400 python -m pytest tests/test_gpu_fuzz.py -q -m gpu -p no:cacheprovider > gpurun_out/r2i_fuzz_campaign.txt 2>&1; echo rc=$? >> gpurun_out/r2i_fuzz_campaign.txt
tail -n 3 gpurun_out/r2i_fuzz_campaign.txt
PGRID_FUZZ_BLOCKS=16 PGRID_LIB=$PWD/paper_2403_10647_b200/_lib/libpgrid_checked.so timeout 2400 python -m pytest tests/test_gpu_fuzz.py -q -m gpu -p no:cacheprovider > gpurun_out/r2i_fuzz_campaign_checked.txt 2>&1; echo rc=$? >> gpurun_out/r2i_fuzz_campaign_checked.txt
tail -n 3 gpurun_out/r2i_fuzz_campaign_checked.txt
