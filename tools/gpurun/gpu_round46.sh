#!/bin/bash
# refine with Y_i widened to double in shared memory (one F2F per element) vs
# the previous float staging (ACCORD_REFINE_YF=1); parity suite first.
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -m gpu -x -q > gpurun_out/pytest_gpu46.log 2>&1; echo pt=$?
for i in 1 2; do
for c in 3 4; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/b46_c${c}_yd_$i.json 2>gpurun_out/b46_c${c}_yd_$i.log
  ACCORD_REFINE_YF=1 timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/b46_c${c}_yf_$i.json 2>gpurun_out/b46_c${c}_yf_$i.log
done
done
timeout 600 python bench.py --config 5 --no-e2e --no-cpu-baseline > gpurun_out/b46_c5_yd.json 2>gpurun_out/b46_c5_yd.log
ACCORD_REFINE_YF=1 timeout 600 python bench.py --config 5 --no-e2e --no-cpu-baseline > gpurun_out/b46_c5_yf.json 2>gpurun_out/b46_c5_yf.log
tail -2 gpurun_out/pytest_gpu46.log
