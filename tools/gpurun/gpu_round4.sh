set -x
timeout 900 python -m pytest tests/test_multirank.py tests/test_gpu_next.py -m gpu -q > gpurun_out/pytest_gpu4.log 2>&1; echo pytest=$?
timeout 900 python tools/gemm_sweep.py 5 0,32 0,16 0,24 0,32,8 0,32,16 2,32 > gpurun_out/sweep4.log 2>&1; echo sweep=$?
tail -3 gpurun_out/pytest_gpu4.log
