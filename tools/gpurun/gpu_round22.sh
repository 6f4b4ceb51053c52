timeout 900 python tools/gemm_power.py 5 > gpurun_out/power22.log 2>&1; echo p=$?
