set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -m gpu -x -q > gpurun_out/pytest_gpu15.log 2>&1; echo pytest=$?
ACCORD_TRACE=1 timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench15_tma.json 2> gpurun_out/bench15_tma.log; echo b1=$?
tail -3 gpurun_out/pytest_gpu15.log
