# Round 2c: c6 / c4 SpMM A-B (the final set showed c6's SpMM at 1.15 ms per
# step against 0.47 at head): previous commit's library vs the final build at
# 8 / 16 ring stages.
set -x
mkdir -p gpurun_out
for c in 6 4; do
for v in nest2 s8 s16; do
  case $v in nest2) E="ACCORD_LIB=$PWD/paper_2412_11554_b200/libaccord_nest2.so";; s8) E="ACCORD_SPMM_STAGES=8";; s16) E="ACCORD_SPMM_STAGES=16";; esac
  env $E timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c6ab_c${c}_$v.json 2> gpurun_out/c6ab_c${c}_$v.log; echo c$c$v=$?
done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/c6ab_launches_c6.csv \
  python bench.py --config 6 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c6ab_ncu_launches.log 2>&1; echo launches=$?
