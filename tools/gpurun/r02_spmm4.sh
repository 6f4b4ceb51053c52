# Round 2, third session: the SpMM's warp-parallel producer issue. GPU tests
# of the SpMM paths, a same-box c5 A-B (parallel vs serial producer issue; 8
# vs 16 ring stages) with the per-phase trace, and an ncu capture of three
# SpMM launches (iteration 2's long rows, the steady state).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "spmm or bitwise or paired" > gpurun_out/s4_pytest.log 2>&1; echo pt=$?
for rep in 1 2; do
for v in par serial par16; do
  case $v in serial) E="ACCORD_SPMM_SERIAL=1";; par16) E="ACCORD_SPMM_STAGES=16";; *) E="";; esac
  env $E ACCORD_TRACE=1 timeout 900 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/s4_${v}_$rep.json 2> gpurun_out/s4_${v}_$rep.log; echo $v$rep=$?
done; done
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:spmm_tma -s 4 -c 4 \
  -o gpurun_out/s4_spmm_c5 -f python bench.py --steps 1 --warmup 4 --no-e2e --no-cpu-baseline > gpurun_out/s4_ncu.log 2>&1; echo ncu=$?
