# Round 2c: why the paired SpMM is slower at c6 (one entry per row) since the
# nested-loop consumer: ncu --set full of the c6 launch, head library vs final.
set -x
mkdir -p gpurun_out
for v in head final; do
  case $v in head) E="ACCORD_LIB=$PWD/paper_2412_11554_b200/libaccord_head.so";; final) E="ACCORD_TRACE=0";; esac
  env $E timeout 600 ncu --set full --import-source on --clock-control none -k 'regex:spmm_tma' -s 4 -c 1 \
    -o gpurun_out/c6ncu_$v -f python bench.py --config 6 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c6ncu_$v.log 2>&1; echo $v=$?
done
