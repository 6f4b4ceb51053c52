# Round 2, second GPU call: lambda_max exactness fix + workspace tests, the
# gather ceiling microbenchmark, an ncu capture of the c5 sparse kernels, and
# bench lines for c3 (L2 flushed), c4, c6.
set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/gather_bench.cu -o /tmp/gather_bench && \
  timeout 300 /tmp/gather_bench > gpurun_out/r02b_gather_bench.txt 2>&1; echo gather=$?
timeout 1200 python -m pytest tests/test_gpu_filter.py -q -k "lambda_max or path" --durations=5 > gpurun_out/r02b_lmax.log 2>&1; echo lmax=$?
timeout 900 python -m pytest tests/test_gpu_workspace.py -q --durations=5 > gpurun_out/r02b_ws.log 2>&1; echo ws=$?
for c in 3 4 6; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/r02b_bench_c$c.json 2> gpurun_out/r02b_bench_c$c.log; echo b$c=$?; done
timeout 1200 ncu --set full --import-source on --clock-control none -k 'regex:spmm_tma|refine_kernel' -s 6 -c 4 \
  -o gpurun_out/r02b_sparse_c5 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02b_ncu_sparse.log 2>&1; echo ncu=$?
