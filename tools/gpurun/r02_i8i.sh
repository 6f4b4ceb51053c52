# Cost check against the support (c3 back to bf16 after one int8 GEMM):
# int8 tests, c3/c5/c6 lines (traced, e2e with create time), then the int8
# GEMM group-size sweep and epilogue share.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_i8.py > gpurun_out/i8i_pytest.log 2>&1; echo pt=$?
for c in 3 6 5; do
  ACCORD_TRACE=1 timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/i8i_c$c.json 2> gpurun_out/i8i_c$c.log; echo b$c=$?
done
bash tools/gpurun/r02_gemm_i8.sh
