# Line-search pass pairing A-B at c5 (same box, alternating): paired passes
# (default) vs one step size per pass (ACCORD_LS_PAIRS=0); e2e included.
set -x
mkdir -p gpurun_out
for rep in 1 2; do for k in 1 0; do
  ACCORD_LS_PAIRS=$k ACCORD_TRACE=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/pairs_c5_${k}_$rep.json 2> gpurun_out/pairs_c5_${k}_$rep.log; echo p$k$rep=$?
done; done
