# Round 2, third session: SpMM consumer rework (one staged row per round,
# accumulators in place, row finalize at the loop top; warp-parallel producer
# issue). GPU tests of the SpMM paths and parity, then a same-box c5 A-B with
# the per-phase trace: the HEAD library, the two-stage consumer
# (ACCORD_SPMM_TWOSTAGE build) and the product; ncu of four SpMM launches.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "spmm or bitwise or paired or f32_small or config2 or dense" > gpurun_out/s5_pytest.log 2>&1; echo pt=$?
for rep in 1 2; do
for v in head two one; do
  case $v in head) E="ACCORD_LIB=$PWD/ab_libs/libaccord_head.so";; two) E="ACCORD_LIB=$PWD/ab_libs/libaccord_twostage.so";; *) E="";; esac
  env $E ACCORD_TRACE=1 timeout 900 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/s5_${v}_$rep.json 2> gpurun_out/s5_${v}_$rep.log; echo $v$rep=$?
done; done
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:spmm_tma -s 4 -c 4 \
  -o gpurun_out/s5_spmm_c5 -f python bench.py --steps 1 --warmup 4 --no-e2e --no-cpu-baseline > gpurun_out/s5_ncu.log 2>&1; echo ncu=$?
