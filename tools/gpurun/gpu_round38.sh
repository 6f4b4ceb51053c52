timeout 900 python bench.py > gpurun_out/b38_c5.json 2> gpurun_out/b38_c5.log; echo b5=$?
timeout 1500 python -m pytest tests/test_gpu_next.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/pytest_gpu38.log 2>&1; echo pt=$?
tail -2 gpurun_out/pytest_gpu38.log
