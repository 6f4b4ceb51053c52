timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -m gpu -x -q > gpurun_out/pytest_gpu26.log 2>&1; echo pytest=$?
timeout 900 python tools/gemm_power.py 5 0,5,0 > gpurun_out/power26.log 2>&1; echo p=$?
tail -2 gpurun_out/pytest_gpu26.log
