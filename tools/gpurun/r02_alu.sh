# Refine A-B: Y_i converted to double on the integer pipe (ACCORD_REFINE=alu)
# vs F2F (default), same box, alternating; parity of the ALU variant.
set -x
mkdir -p gpurun_out
ACCORD_REFINE=alu timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "config2 or small or refit or dense or beyond or reproducible" > gpurun_out/alu_tests.log 2>&1; echo t=$?
for rep in 1 2; do for k in block alu; do
  ACCORD_REFINE=$k timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/alu_c5_${k}_$rep.json 2> /dev/null; echo c5$k$rep=$?
  ACCORD_REFINE=$k timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/alu_c3_${k}_$rep.json 2> /dev/null; echo c3$k$rep=$?
done; done
