# Operand width A-B at c5 (same box, alternating): full bf16 vs mantissa bits
# dropped from the X^T_hi / Y_hi GEMM operands once |C| / p <= 64; then the
# filter certification and the config-3 full-oracle schedule with the narrow
# operands from iteration 2 on (ACCORD_XDROP_AT huge).
set -x
mkdir -p gpurun_out
for rep in 1 2; do for xy in 0_0 1_1 1_0 2_1; do
  x=${xy%_*}; y=${xy#*_}
  ACCORD_XDROP=$x ACCORD_YDROP=$y timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/xydrop_c5_${xy}_$rep.json 2> gpurun_out/xydrop_c5_${xy}_$rep.log; echo x$xy$rep=$?
done; done
ACCORD_XDROP=1 ACCORD_YDROP=1 ACCORD_XDROP_AT=1e12 timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_filter.py > gpurun_out/xydrop_pytest_filter.log 2>&1; echo pf=$?
ACCORD_XDROP=1 ACCORD_YDROP=1 ACCORD_XDROP_AT=1e12 timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_fullsize.py -k config3_full_oracle > gpurun_out/xydrop_pytest_c3.log 2>&1; echo pc=$?
