set -x
ACCORD_TRACE=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench11.json 2> gpurun_out/bench11_trace.log; echo bench=$?
timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain11.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:spmm_kernel|refine_kernel' -s 8 -c 3 -o gpurun_out/prof_sparse_c5 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu11.log 2>&1; echo ncu=$?
