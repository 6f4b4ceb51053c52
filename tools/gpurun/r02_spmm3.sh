# Round 2, third session: the SpMM's barrier-free row finalize. GPU tests of
# the SpMM paths, then a same-box c5 A-B (block barrier per row vs
# barrier-free; register budget 3 vs 2 blocks per SM) with the per-phase
# trace (iteration 2's long rows and the steady state), and an ncu capture of
# the paired SpMM (stall reasons by source line).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "spmm or bitwise or paired" > gpurun_out/s3_pytest.log 2>&1; echo pt=$?
for rep in 1 2; do
for v in nobar bar minb2; do
  case $v in bar) E="ACCORD_SPMM_BAR=1";; minb2) E="ACCORD_SPMM_MINB=2";; *) E="";; esac
  env $E ACCORD_TRACE=1 timeout 900 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/s3_${v}_$rep.json 2> gpurun_out/s3_${v}_$rep.log; echo $v$rep=$?
done; done
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:spmm_tma -s 12 -c 2 \
  -o gpurun_out/s3_spmm_c5 -f python bench.py --steps 1 --warmup 4 --no-e2e --no-cpu-baseline > gpurun_out/s3_ncu.log 2>&1; echo ncu=$?
