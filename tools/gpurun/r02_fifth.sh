# Round 2, fifth GPU call: SpMM 4 vs 8 columns per consumer thread, refine
# block sizes, create-time trace, parity of the SpMM variants.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tma_spmm or paired or first_iteration or parity_f32_small" > gpurun_out/r02e_parity.log 2>&1; echo par=$?
for c in 3 5; do
  for cols in 4 8; do
    ACCORD_REFINE=block ACCORD_SPMM_COLS=$cols timeout 900 python bench.py --config $c --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02e_bench_c${c}_cols$cols.json 2> gpurun_out/r02e_bench_c${c}_cols$cols.log; echo b$c$cols=$?
  done
  for t in 64 128; do
    ACCORD_REFINE=block ACCORD_REFINE_THREADS=$t timeout 900 python bench.py --config $c --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02e_bench_c${c}_thr$t.json 2> gpurun_out/r02e_bench_c${c}_thr$t.log; echo b$c$t=$?
  done
done
ACCORD_TRACE=1 timeout 900 python tools/create_timing.py 5 > gpurun_out/r02e_create.log 2>&1; echo create=$?
