#!/bin/bash
# ncu --set full of the c5 sparse kernels (TMA SpMM, refine) on the final build
set -x
timeout 600 python bench.py --steps 1 --warmup 4 --no-e2e --no-cpu-baseline > gpurun_out/b52_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:spmm_tma|refine_kernel' -s 7 -c 3 \
  -o gpurun_out/final_prof_sparse_c5 -f python bench.py --steps 1 --warmup 4 --no-e2e --no-cpu-baseline > gpurun_out/ncu52.log 2>&1
echo ncu=$?
