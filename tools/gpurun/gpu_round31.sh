set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -m gpu -x -q > gpurun_out/pytest_gpu31.log 2>&1; echo pytest=$?
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "4 or 5" > gpurun_out/pytest_gpu31b.log 2>&1; echo pytest2=$?
ACCORD_TRACE=1 timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/b31_pairs.json 2> gpurun_out/b31_pairs.log; echo b1=$?
ACCORD_LS_PAIRS=0 timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/b31_seq.json 2> gpurun_out/b31_seq.log; echo b2=$?
tail -3 gpurun_out/pytest_gpu31.log; tail -3 gpurun_out/pytest_gpu31b.log
