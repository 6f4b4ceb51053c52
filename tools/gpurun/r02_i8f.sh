# int8 cost check (off for the solve when int8 adds > 5e-4 p^2 candidates):
# all GPU tests, c3 traced (bench + e2e), c5 line.
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/i8f_pytest_all.log 2>&1; echo all=$?
ACCORD_TRACE=1 timeout 900 python bench.py --config 3 --no-cpu-baseline > gpurun_out/i8f_c3.json 2> gpurun_out/i8f_c3.log; echo b3=$?
timeout 900 python bench.py --config 4 --no-cpu-baseline > gpurun_out/i8f_c4.json 2> gpurun_out/i8f_c4.log; echo b4=$?
timeout 900 python bench.py > gpurun_out/i8f_c5.json 2> gpurun_out/i8f_c5.log; echo b5=$?
