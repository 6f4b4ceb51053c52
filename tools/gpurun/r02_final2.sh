# Round-2 final set on the int8-filter build: all GPU tests, smoke, parity
# report (AUTO), bench lines (c5 with cpu_baseline + e2e, reference arm,
# c3/c4/c6), the ncu launch list of the c5 bench command, ncu --set full of
# one steady-state int8 GEMM and of the steady-state sparse kernels.
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/f2_pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/f2_bench_c5.json 2> gpurun_out/f2_bench_c5.log; echo b5=$?
timeout 1200 python bench.py --impl reference > gpurun_out/f2_reference_c5.json 2> gpurun_out/f2_reference_c5.log; echo ref=$?
for c in 3 4 6; do timeout 900 python bench.py --config $c > gpurun_out/f2_bench_c$c.json 2> gpurun_out/f2_bench_c$c.log; echo b$c=$?; done
timeout 2400 python tools/parity_report.py > gpurun_out/f2_parity_report.json 2> gpurun_out/f2_parity_report.log; echo parity=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f2_launches_c5.csv \
  python bench.py --steps 2 --warmup 4 --no-e2e --no-cpu-baseline > gpurun_out/f2_ncu_launches.log 2>&1; echo launches=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 5 -c 1 \
  -o gpurun_out/f2_gemm_c5 -f python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/f2_ncu_gemm.log 2>&1; echo ncugemm=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k 'regex:spmm_tma|refine_kernel' -s 9 -c 3 \
  -o gpurun_out/f2_sparse_c5 -f python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/f2_ncu_sparse.log 2>&1; echo ncusparse=$?
