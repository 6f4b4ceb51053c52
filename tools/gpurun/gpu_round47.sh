#!/bin/bash
# (1) per-phase trace of the first c5 iterations (e2e cost of iterations 1-3)
# (2) ncu --set full of the c3 refine and SpMM (L2-resident X^T: what bounds them)
set -x
ACCORD_TRACE=1 timeout 600 python bench.py --config 5 --warmup 3 --steps 1 --no-e2e --no-cpu-baseline > gpurun_out/b47_c5_trace.json 2> gpurun_out/b47_c5_trace.log
timeout 300 python bench.py --config 3 --warmup 3 --steps 2 --no-e2e --no-cpu-baseline > gpurun_out/b47_c3.json 2> gpurun_out/b47_c3.log && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"refine_kernel|spmm_kernel" -s 20 -c 2 \
  -o gpurun_out/ncu47_c3_sparse -f python bench.py --config 3 --warmup 3 --steps 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu47.log 2>&1
echo ncu=$?
