timeout 900 python tools/create_timing.py 5 > gpurun_out/create35.log 2>&1; echo c=$?
