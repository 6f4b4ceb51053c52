# Paired SpMM: producer lookahead of two items (default now) A-B'd against
# register budget for 2 blocks (no spills); parity subset; ncu of the pass.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "paired or config2_full or bitwise" > gpurun_out/sp_pytest.log 2>&1; echo pt=$?
for rep in 1 2; do for m in 0 2; do
  ACCORD_SPMM_MINB=$m timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/sp_c5_minb${m}_$rep.json 2> gpurun_out/sp_c5_minb${m}_$rep.log; echo b$m$rep=$?
done; done
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:spmm_tma -s 8 -c 2 \
  -o gpurun_out/sp_spmm_c5 -f python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/sp_ncu.log 2>&1; echo ncu=$?
