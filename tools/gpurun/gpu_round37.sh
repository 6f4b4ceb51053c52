timeout 900 python tools/create_timing.py 5 > gpurun_out/create37.log 2>&1; echo c=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sample_major or errors or objective" > gpurun_out/pytest_gpu37.log 2>&1; echo pt=$?
tail -2 gpurun_out/pytest_gpu37.log
