# SpMM without the bf16 operand while the int8 GEMM is on (A-B vs
# ACCORD_SPMM_BF16=1, same box), int8 + parity tests, and a source-level ncu
# of the steady-state paired SpMM.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_i8.py tests/test_gpu_parity.py > gpurun_out/i8g_pytest.log 2>&1; echo pt=$?
for rep in 1 2; do for k in 0 1; do
  ACCORD_SPMM_BF16=$k timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/i8g_c5_bf16spmm${k}_$rep.json 2> gpurun_out/i8g_c5_bf16spmm${k}_$rep.log; echo b$k$rep=$?
done; done
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:spmm_tma -s 8 -c 2 \
  -o gpurun_out/i8g_spmm_c5 -f python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/i8g_ncu_spmm.log 2>&1; echo ncu=$?
