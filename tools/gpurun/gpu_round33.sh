SWEEP_REPS=6 timeout 1200 python tools/gemm_sweep.py 5 0,32 0,48 0,64 > gpurun_out/sweep33_c5.log 2>&1; echo s5=$?
timeout 1200 python -m pytest tests/test_multirank.py -m gpu -x -q -k "p_invariance" > gpurun_out/pytest_gpu33.log 2>&1; echo pt=$?
tail -2 gpurun_out/pytest_gpu33.log
