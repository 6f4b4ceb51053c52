# refine with Y_i staged as float64 (one F2F per product) + the nnz-based
# int8 switch: all GPU tests, c5 line (cpu_baseline, e2e), refine A-B vs the
# f32-staged refine, c3/c4/c6 lines.
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/i8e_pytest_all.log 2>&1; echo all=$?
ACCORD_TRACE=1 timeout 900 python bench.py > gpurun_out/i8e_c5.json 2> gpurun_out/i8e_c5.log; echo b5=$?
ACCORD_REFINE=f32 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/i8e_c5_reff32.json 2> gpurun_out/i8e_c5_reff32.log; echo b5r=$?
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/i8e_c5_refd.json 2> gpurun_out/i8e_c5_refd.log; echo b5d=$?
for c in 3 4 6; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/i8e_c$c.json 2> gpurun_out/i8e_c$c.log; echo b$c=$?
done
