# AUTO's adaptive int8 switch on the other configs (c3, c4, c6: auto vs bf16,
# same box), the c5 bench line with cpu_baseline, its ncu launch list, and an
# ncu --set full of one steady-state int8 GEMM (5th GEMM launch: iterations
# 1-3 run bf16).
set -x
mkdir -p gpurun_out
for c in 3 4 6; do for g in auto bf16; do
  ACCORD_AUTO_GEMM=$g timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/i8c_c${c}_$g.json 2> gpurun_out/i8c_c${c}_$g.log; echo b$c$g=$?
done; done
timeout 900 python bench.py > gpurun_out/i8c_c5.json 2> gpurun_out/i8c_c5.log; echo b5=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/i8c_launches_c5.csv \
  python bench.py --steps 2 --warmup 4 --no-e2e --no-cpu-baseline > gpurun_out/i8c_ncu_launches.log 2>&1; echo launches=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 5 -c 1 \
  -o gpurun_out/i8c_gemm_c5 -f python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/i8c_ncu_gemm.log 2>&1; echo ncugemm=$?
