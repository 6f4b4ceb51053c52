#!/bin/bash
# symmetric first GEMM (Omega = I): bitwise test, parity suites, c5 trace + e2e
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k symmetric > gpurun_out/pytest_gpu48_sym.log 2>&1; echo sym=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu48.log 2>&1; echo pt=$?
ACCORD_TRACE=1 timeout 600 python bench.py --config 5 --warmup 3 --steps 5 --no-cpu-baseline > gpurun_out/b48_c5.json 2> gpurun_out/b48_c5.log
ACCORD_GEMM_NOSYM=1 timeout 600 python bench.py --config 5 --warmup 3 --steps 5 --no-cpu-baseline > gpurun_out/b48_c5_nosym.json 2> gpurun_out/b48_c5_nosym.log
tail -2 gpurun_out/pytest_gpu48.log
