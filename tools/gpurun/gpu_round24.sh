timeout 900 python tools/gemm_power.py 5 0,4,3,0 > gpurun_out/power24.log 2>&1; echo p=$?
