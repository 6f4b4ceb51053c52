# ncu of the paired SpMM pass of iteration 2 (long rows: 2.4e8 entries) and
# of the unpaired z pass of iteration 1, source-level, to find what holds
# the paired kernel at half the unpaired one's bandwidth.
set -x
mkdir -p gpurun_out
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:spmm_tma -s 1 -c 2 \
  -o gpurun_out/pair_spmm_c5 -f python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/pair_ncu.log 2>&1; echo ncu=$?
