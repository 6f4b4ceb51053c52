# Round 2, ninth GPU call: product GEMM without the multi-rank mirror branch
# (kDiag 3 variant for sym 2), grouped refine (A-B vs block), parity.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_multirank.py tests/test_gpu_parity.py -q -x -m gpu -k "symmetric or invariance or reproducible or config2 or beyond" > gpurun_out/r02i_tests.log 2>&1; echo tests=$?
ACCORD_REFINE=group timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "config2 or small or refit or dense or beyond or reproducible" > gpurun_out/r02i_tests_group.log 2>&1; echo tgroup=$?
for rep in 1 2; do
  for k in block group; do
    ACCORD_REFINE=$k timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02i_bench_c5_${k}_$rep.json 2> gpurun_out/r02i_bench_c5_${k}_$rep.log; echo c5$k$rep=$?
  done
done
for k in block group; do
  ACCORD_REFINE=$k timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02i_bench_c3_$k.json 2> gpurun_out/r02i_bench_c3_$k.log; echo c3$k=$?
  ACCORD_REFINE=$k timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02i_bench_c4_$k.json 2> gpurun_out/r02i_bench_c4_$k.log; echo c4$k=$?
done
