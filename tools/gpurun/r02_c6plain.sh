# Round 2c: c6 with the block-per-row SpMM (ACCORD_SPMM_PLAIN=1) vs the TMA
# kernel: a measurement for the next round's routing rule, no code change.
set -x
mkdir -p gpurun_out
for v in tma plain; do
  case $v in tma) E="ACCORD_TRACE=0";; plain) E="ACCORD_SPMM_PLAIN=1";; esac
  env $E timeout 300 python bench.py --config 6 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c6plain_$v.json 2> gpurun_out/c6plain_$v.log; echo $v=$?
done
