set -x
timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain16.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:spmm_tma|refine_kernel' -s 6 -c 4 -o gpurun_out/prof_sparse16 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu16.log 2>&1; echo ncu=$?
