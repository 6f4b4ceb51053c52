timeout 900 python tools/gemm_power.py 5 0,5,6,0 > gpurun_out/power25.log 2>&1; echo p=$?
