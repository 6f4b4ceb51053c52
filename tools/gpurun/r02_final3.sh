# Round 2c final set (reworked TMA SpMM: nested-loop branch-free consumer,
# two-batch item lookahead, 16 stages): all GPU tests, smoke, bench lines (c5
# with cpu_baseline + e2e, c3/c4/c6), same-box SpMM A-B against the previous
# commit's library, the ncu launch list of the c5 bench command, ncu --set full
# of the steady-state sparse kernels, parity report.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/f3_pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/f3_bench_c5.json 2> gpurun_out/f3_bench_c5.log; echo b5=$?
for c in 3 4 6; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/f3_bench_c$c.json 2> gpurun_out/f3_bench_c$c.log; echo b$c=$?; done
for rep in 1 2; do
for v in nest2 final; do
  case $v in nest2) E="ACCORD_LIB=$PWD/paper_2412_11554_b200/libaccord_nest2.so";; final) E="ACCORD_TRACE=1";; esac
  env $E timeout 900 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/f3_ab_${v}_$rep.json 2> gpurun_out/f3_ab_${v}_$rep.log; echo $v$rep=$?
done; done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f3_launches_c5.csv \
  python bench.py --steps 2 --warmup 4 --no-e2e --no-cpu-baseline > gpurun_out/f3_ncu_launches.log 2>&1; echo launches=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k 'regex:spmm_tma|refine_kernel' -s 9 -c 3 \
  -o gpurun_out/f3_sparse_c5 -f python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/f3_ncu_sparse.log 2>&1; echo ncusparse=$?
timeout 900 python tools/parity_report.py > gpurun_out/f3_parity_report.json 2> gpurun_out/f3_parity_report.log; echo parity=$?
