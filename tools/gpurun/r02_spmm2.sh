# Paired SpMM producer: raw metadata loads converted at use, item map one
# batch ahead; parity subset + c5 line + ncu of the pass; then the int8-from-
# iteration-2 run (r02_i8h.sh).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "paired or config2_full or bitwise or dense_candidate" > gpurun_out/sp2_pytest.log 2>&1; echo pt=$?
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/sp2_c5.json 2> gpurun_out/sp2_c5.log; echo b5=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:spmm_tma -s 8 -c 2 \
  -o gpurun_out/sp2_spmm_c5 -f python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/sp2_ncu.log 2>&1; echo ncu=$?
bash tools/gpurun/r02_i8h.sh
