# int8 from iteration 2 (nnz/p <= 256 after iteration 1): c5 traced line with
# e2e, c3/c4/c6, int8 + parity tests.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_i8.py tests/test_gpu_parity.py > gpurun_out/i8h_pytest.log 2>&1; echo pt=$?
ACCORD_TRACE=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/i8h_c5.json 2> gpurun_out/i8h_c5.log; echo b5=$?
for c in 3 4 6; do
  ACCORD_TRACE=1 timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/i8h_c$c.json 2> gpurun_out/i8h_c$c.log; echo b$c=$?
done
