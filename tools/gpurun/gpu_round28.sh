set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py tests/test_multirank.py -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu28.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/b28_c5.json 2> gpurun_out/b28_c5.log; echo b5=$?
tail -2 gpurun_out/pytest_gpu28.log
