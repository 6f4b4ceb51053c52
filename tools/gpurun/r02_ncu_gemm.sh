# ncu --set full of one steady-state c5 GEMM launch (the 5th: iterations 1-4
# are the warm-up) for roofline.traffic; c4 create-phase trace (e2e noise).
set -x
mkdir -p gpurun_out
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 4 -c 1 \
  -o gpurun_out/fin_gemm_c5 -f python bench.py --steps 1 --warmup 4 --no-e2e --no-cpu-baseline > gpurun_out/fin_ncu_gemm.log 2>&1; echo ncugemm=$?
ACCORD_TRACE=1 timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02l_bench_c4.json 2> gpurun_out/r02l_bench_c4.log; echo b4=$?
