timeout 900 python tools/gemm_sweep.py 5 0,32 0,24 0,48 0,16 > gpurun_out/sweep32_c5.log 2>&1; echo s5=$?
timeout 900 python tools/gemm_sweep.py 4 0,32 0,16 0,8 0,24 > gpurun_out/sweep32_c4.log 2>&1; echo s4=$?
