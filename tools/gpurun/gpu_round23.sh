timeout 900 python tools/gemm_power.py 5 0,1,3,4,0 > gpurun_out/power23.log 2>&1; echo p=$?
