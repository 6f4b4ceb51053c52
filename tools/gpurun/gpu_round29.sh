set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -m gpu -x -q > gpurun_out/pytest_gpu29.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/b29_c5.json 2> gpurun_out/b29_c5.log; echo b5=$?
tail -5 gpurun_out/pytest_gpu29.log
