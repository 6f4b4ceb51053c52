set -x
timeout 900 python -m pytest tests/test_multirank.py tests/test_gpu_next.py -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; echo pytest=$?
timeout 900 python tools/gemm_sweep.py 5 --kfull 0,64 1,64 2,64 0,32 > gpurun_out/sweep3.log 2>&1; echo sweep=$?
tail -3 gpurun_out/pytest_gpu3.log
