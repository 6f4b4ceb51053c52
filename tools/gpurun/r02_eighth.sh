# Round 2, eighth GPU call: SpMM one barrier per row; same-box A-B of the
# epilogue with / without the multi-rank mirror branch (ACCORD_NO_SYM2 build),
# alternating; the reference arm next to our cpu_baseline.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tma_spmm or paired or reproducible or config2" > gpurun_out/r02h_parity.log 2>&1; echo par=$?
for rep in 1 2; do
  timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02h_bench_c5_main$rep.json 2> gpurun_out/r02h_bench_c5_main$rep.log; echo main$rep=$?
  ACCORD_LIB=paper_2412_11554_b200/libaccord_nosym2.so timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02h_bench_c5_nosym2_$rep.json 2> gpurun_out/r02h_bench_c5_nosym2_$rep.log; echo nosym2_$rep=$?
done
timeout 1200 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02h_reference_c5.json 2> gpurun_out/r02h_reference_c5.log; echo ref=$?
