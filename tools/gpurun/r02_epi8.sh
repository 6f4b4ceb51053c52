# int8 GEMM with 8 epilogue warps (two per TMEM lane quarter) and the refine's
# conflict-free float64 staging: int8 + parity tests, c5 line, c3 line.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_i8.py tests/test_gpu_parity.py > gpurun_out/e8_pytest.log 2>&1; echo pt=$?
ACCORD_TRACE=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/e8_c5.json 2> gpurun_out/e8_c5.log; echo b5=$?
timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/e8_c3.json 2> gpurun_out/e8_c3.log; echo b3=$?
ACCORD_REFINE=f32 timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/e8_c3_reff32.json 2> gpurun_out/e8_c3_reff32.log; echo b3f=$?
ACCORD_DEBUG_GEMM=1 timeout 900 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/e8_noepi.json 2> gpurun_out/e8_noepi.log; echo noepi=$?
