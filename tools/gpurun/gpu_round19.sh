set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -m gpu -x -q > gpurun_out/pytest_gpu19.log 2>&1; echo pytest=$?
timeout 600 python bench.py --config 3 --no-e2e --no-cpu-baseline > gpurun_out/b19_c3.json 2>/dev/null; echo c3=$?
ACCORD_FILTER_EXACT=1 timeout 600 python bench.py --config 3 --no-e2e --no-cpu-baseline > gpurun_out/b19_c3_exact.json 2>/dev/null; echo c3x=$?
timeout 600 python bench.py --config 4 --no-e2e --no-cpu-baseline > gpurun_out/b19_c4.json 2>/dev/null; echo c4=$?
ACCORD_FILTER_EXACT=1 timeout 600 python bench.py --config 4 --no-e2e --no-cpu-baseline > gpurun_out/b19_c4_exact.json 2>/dev/null; echo c4x=$?
timeout 900 python tools/gemm_sweep.py 5 0,32 > gpurun_out/sweep19.log 2>&1; echo s=$?
ACCORD_FILTER_EXACT=1 timeout 900 python tools/gemm_sweep.py 5 0,32 > gpurun_out/sweep19_exact.log 2>&1; echo sx=$?
tail -2 gpurun_out/pytest_gpu19.log
