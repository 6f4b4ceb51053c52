set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -m gpu -x -q -k "not dense_candidate" > gpurun_out/pytest_gpu5.log 2>&1; echo pytest=$?
timeout 600 python tools/gemm_sweep.py 5 0,32 0,64 > gpurun_out/sweep5_elect.log 2>&1; echo sweep=$?
ACCORD_LIB=$PWD/paper_2412_11554_b200/libaccord_lane0.so timeout 600 python tools/gemm_sweep.py 5 0,32 0,64 > gpurun_out/sweep5_lane0.log 2>&1; echo sweep=$?
timeout 600 python tools/gemm_sweep.py 5 0,32 0,64 > gpurun_out/sweep5_elect_b.log 2>&1; echo sweep=$?
tail -3 gpurun_out/pytest_gpu5.log
