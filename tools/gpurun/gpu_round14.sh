set -x
timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain14.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:spmm_tma -s 5 -c 1 -o gpurun_out/prof_spmm_tma python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu14.log 2>&1; echo ncu=$?
