set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_gpu13.log 2>&1; echo pytest=$?
ACCORD_TRACE=1 timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench13_tma.json 2> gpurun_out/bench13_tma.log; echo b1=$?
ACCORD_SPMM_PLAIN=1 ACCORD_TRACE=1 timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench13_plain.json 2> gpurun_out/bench13_plain.log; echo b2=$?
tail -3 gpurun_out/pytest_gpu13.log
