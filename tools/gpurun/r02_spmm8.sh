# Round 2, fifth session: nested-loop consumer with the trimmed inner loop
# (32-bit shared addresses, dataless stages skipped, unused norm reductions
# skipped): SpMM parity tests, same-box A-B against the head library, ncu of
# the sparse kernels.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "spmm or bitwise or paired or f32_small or config2 or dense" > gpurun_out/s8_pytest.log 2>&1; echo pt=$?
for rep in 1 2; do
for v in head nest nest2; do
  case $v in head) E="ACCORD_LIB=$PWD/paper_2412_11554_b200/libaccord_head.so";; nest) E="ACCORD_LIB=$PWD/paper_2412_11554_b200/libaccord_nest.so";; nest2) E="ACCORD_SPMM_STAGES=8";; esac
  env $E ACCORD_TRACE=1 timeout 900 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/s8_${v}_$rep.json 2> gpurun_out/s8_${v}_$rep.log; echo $v$rep=$?
done; done
timeout 1500 ncu --set full --import-source on --clock-control none -k 'regex:spmm_tma' -s 6 -c 2 \
  -o gpurun_out/s8_sparse_c5 -f python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/s8_ncu_sparse.log 2>&1; echo ncusparse=$?
