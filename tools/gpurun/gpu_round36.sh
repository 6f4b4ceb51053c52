set -x
timeout 900 python tools/create_timing.py 5 > gpurun_out/create36.log 2>&1; echo c=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_multirank.py -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu36.log 2>&1; echo pt=$?
timeout 900 python bench.py > gpurun_out/b36_c5.json 2> gpurun_out/b36_c5.log; echo b5=$?
tail -3 gpurun_out/pytest_gpu36.log
