#!/bin/bash
# c3 (p = 2e4, below the TMA SpMM row threshold): block-per-row vs TMA SpMM
for i in 1 2; do
  timeout 300 python bench.py --config 3 --no-e2e --no-cpu-baseline > gpurun_out/b54_c3_plain_$i.json 2>/dev/null
  ACCORD_SPMM_TMA=1 timeout 300 python bench.py --config 3 --no-e2e --no-cpu-baseline > gpurun_out/b54_c3_tma_$i.json 2>/dev/null
done
