set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_gpu43.log 2>&1; echo pt=$?
for i in 1 2; do
timeout 600 python bench.py --config 6 --no-e2e --no-cpu-baseline > gpurun_out/b43_c6_new$i.json 2>/dev/null
ACCORD_LIB=$PWD/paper_2412_11554_b200/libaccord_prev.so timeout 600 python bench.py --config 6 --no-e2e --no-cpu-baseline > gpurun_out/b43_c6_prev$i.json 2>/dev/null
done
timeout 900 python tools/gemm_sweep.py 5 0,48 > gpurun_out/sweep43_new.log 2>&1
ACCORD_LIB=$PWD/paper_2412_11554_b200/libaccord_prev.so timeout 900 python tools/gemm_sweep.py 5 0,48 > gpurun_out/sweep43_prev.log 2>&1
tail -2 gpurun_out/pytest_gpu43.log
