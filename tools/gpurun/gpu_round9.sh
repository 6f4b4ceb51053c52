set -x
timeout 900 python tools/gemm_sweep.py 4 0,32,0 0,16,0 0,16,4 0,16,8 0,8,0 0,8,4 > gpurun_out/sweep9_c4.log 2>&1; echo s4=$?
timeout 900 python tools/gemm_sweep.py 5 0,32,0 0,32,8 0,16,4 0,32,16 0,16,8 > gpurun_out/sweep9_c5.log 2>&1; echo s5=$?
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain9.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 450 -c 300 --csv --log-file gpurun_out/launches_c5_v9.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu9.log 2>&1; echo ncu=$?
