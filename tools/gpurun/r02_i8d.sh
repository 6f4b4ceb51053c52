# int8 X^T with the variables permuted by max |x| (block scale ~ per-variable
# scale): int8 tests, c5/c4/c6 bench (traced), refine block-size A-B at c5.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_i8.py > gpurun_out/i8d_pytest.log 2>&1; echo pt=$?
ACCORD_TRACE=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/i8d_c5.json 2> gpurun_out/i8d_c5.log; echo b5=$?
for c in 4 6; do
  ACCORD_TRACE=1 timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/i8d_c$c.json 2> gpurun_out/i8d_c$c.log; echo b$c=$?
done
ACCORD_REFINE_THREADS=256 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/i8d_c5_thr256.json 2> gpurun_out/i8d_c5_thr256.log; echo b5t=$?
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/i8d_c5_thr128.json 2> gpurun_out/i8d_c5_thr128.log; echo b5t=$?
