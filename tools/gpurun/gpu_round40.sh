timeout 900 python tools/gemm_power.py 6 0,1,0,1 > gpurun_out/power40.log 2>&1; echo p=$?
