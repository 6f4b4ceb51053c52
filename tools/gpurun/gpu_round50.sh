#!/bin/bash
# line search from Omega = I (one SpMM for all trials of iteration 1)
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "identity or symmetric or paired" > gpurun_out/pytest_gpu50_diag.log 2>&1; echo diag=$?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu50.log 2>&1; echo pt=$?
ACCORD_TRACE=1 timeout 600 python bench.py --config 5 --warmup 1 --steps 1 --no-e2e --no-cpu-baseline > gpurun_out/b50_trace.json 2> gpurun_out/b50_trace.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/b50_c5.json 2> gpurun_out/b50_c5.log
ACCORD_LS_NODIAG=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/b50_c5_nodiag.json 2> gpurun_out/b50_c5_nodiag.log
tail -3 gpurun_out/pytest_gpu50.log
