mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_mp.log 2>&1; echo rc=$? >> gpurun_out/pytest_mp.log; tail -15 gpurun_out/pytest_mp.log
