# Round 2, fifth session: branch-free consumer loop (every stage carries a row;
# metadata + columns in five back-to-back 16-byte shared loads): SpMM parity
# tests, same-box A-B: nest2 (previous commit), nest3 (this build) with 8 / 16
# stages, nest3 + the second batch of the next items prefetched.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "spmm or bitwise or paired or f32_small or config2 or dense" > gpurun_out/s9_pytest.log 2>&1; echo pt=$?
for rep in 1 2; do
for v in nest2 nest3 nest3s16 pf2 pf2s16; do
  case $v in nest2) E="ACCORD_LIB=$PWD/paper_2412_11554_b200/libaccord_nest2.so";; nest3) E="ACCORD_SPMM_STAGES=8";; nest3s16) E="ACCORD_SPMM_STAGES=16";;
    pf2) E="ACCORD_LIB=$PWD/paper_2412_11554_b200/libaccord_pf2.so";; pf2s16) E="ACCORD_LIB=$PWD/paper_2412_11554_b200/libaccord_pf2.so ACCORD_SPMM_STAGES=16";; esac
  env $E ACCORD_TRACE=1 timeout 900 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/s9_${v}_$rep.json 2> gpurun_out/s9_${v}_$rep.log; echo $v$rep=$?
done; done
