# Round 2, third session: SpMM knobs on the reworked consumer (same box):
# columns per consumer thread 8 / 4, ring stages 8 / 16 / 4.
set -x
mkdir -p gpurun_out
for rep in 1 2; do
for v in c8s8 c4s8 c8s16 c4s16 c8s4; do
  case $v in c8s8) E="ACCORD_SPMM_COLS=8 ACCORD_SPMM_STAGES=8";; c4s8) E="ACCORD_SPMM_COLS=4 ACCORD_SPMM_STAGES=8";;
    c8s16) E="ACCORD_SPMM_COLS=8 ACCORD_SPMM_STAGES=16";; c4s16) E="ACCORD_SPMM_COLS=4 ACCORD_SPMM_STAGES=16";; c8s4) E="ACCORD_SPMM_COLS=8 ACCORD_SPMM_STAGES=4";; esac
  env $E ACCORD_TRACE=1 timeout 900 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/s6_${v}_$rep.json 2> gpurun_out/s6_${v}_$rep.log; echo $v$rep=$?
done; done
