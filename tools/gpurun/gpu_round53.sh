#!/bin/bash
# SpMM ring depth A-B on the final build (paired passes in the steady state)
for st in 8 12 16 8; do
  ACCORD_SPMM_STAGES=$st timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b53_st${st}_$RANDOM.json 2>/dev/null
done
ls gpurun_out/b53_*
