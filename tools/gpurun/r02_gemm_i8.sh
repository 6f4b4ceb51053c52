# int8 GEMM at c5, same box: X^T group size sweep (GN 48 default / 96 / 144:
# Y re-read from DRAM once per group) and the epilogue's share
# (ACCORD_DEBUG_GEMM=1 skips it; results wrong, timing only).
set -x
mkdir -p gpurun_out
for gn in 48 96 144 48; do
  ACCORD_GEMM_GN=$gn timeout 900 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/gi_gn$gn.json 2> gpurun_out/gi_gn$gn.log; echo gn$gn=$?
done
ACCORD_DEBUG_GEMM=1 timeout 900 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/gi_noepi.json 2> gpurun_out/gi_noepi.log; echo noepi=$?
