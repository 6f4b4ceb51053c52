# Round 2, fifth session: head (51db4ef, reworked TMA SpMM) verification on a
# fresh B200: all GPU tests, smoke, c5 bench line, c3/c4/c6 lines, the ncu
# launch list of the c5 bench command, ncu --set full of the sparse kernels.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/h4_pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h4_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/h4_bench_c5.json 2> gpurun_out/h4_bench_c5.log; echo b5=$?
for c in 3 4 6; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/h4_bench_c$c.json 2> gpurun_out/h4_bench_c$c.log; echo b$c=$?; done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/h4_launches_c5.csv \
  python bench.py --steps 2 --warmup 4 --no-e2e --no-cpu-baseline > gpurun_out/h4_ncu_launches.log 2>&1; echo launches=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k 'regex:spmm_tma|refine_kernel' -s 9 -c 3 \
  -o gpurun_out/h4_sparse_c5 -f python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/h4_ncu_sparse.log 2>&1; echo ncusparse=$?
