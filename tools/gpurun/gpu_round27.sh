timeout 900 python tools/gemm_power.py 5 0,7,8,0 > gpurun_out/power27.log 2>&1; echo p=$?
