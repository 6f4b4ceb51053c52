set -x
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "6" > gpurun_out/pytest_gpu30.log 2>&1; echo pytest=$?
ACCORD_TRACE=1 timeout 900 python bench.py --config 6 > gpurun_out/b30_c6.json 2> gpurun_out/b30_c6.log; echo b6=$?
tail -3 gpurun_out/pytest_gpu30.log
