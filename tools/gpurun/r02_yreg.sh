# Refine A-B: Y_i in registers as float64 (ACCORD_REFINE=yreg) vs default;
# parity of the variant; full GPU suite (watchdog test added); c5 bench with
# the e2e settle.
set -x
mkdir -p gpurun_out
ACCORD_REFINE=yreg timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "config2 or small or refit or reproducible or first_iteration" > gpurun_out/yreg_tests.log 2>&1; echo t=$?
for rep in 1 2; do for k in block yreg; do
  ACCORD_REFINE=$k timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/yreg_c3_${k}_$rep.json 2> /dev/null; echo c3$k$rep=$?
  ACCORD_REFINE=$k timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/yreg_c5_${k}_$rep.json 2> /dev/null; echo c5$k$rep=$?
done; done
timeout 3000 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/yreg_pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/yreg_bench_c5.json 2> gpurun_out/yreg_bench_c5.log; echo b5=$?
