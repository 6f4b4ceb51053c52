# Re-entry check of HEAD (symmetric refine): all GPU tests, smoke, c5 bench,
# and an ncu --set full of the steady-state sparse kernels (refine, SpMM).
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/res_pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/res_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/res_bench_c5.json 2> gpurun_out/res_bench_c5.log; echo b5=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k 'regex:spmm_tma|refine_kernel' -s 6 -c 3 \
  -o gpurun_out/res_sparse_c5 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/res_ncu_sparse.log 2>&1; echo ncusparse=$?
