#!/bin/bash
# A-B: filter-GEMM operands rounded to fewer mantissa bits (diagnostic builds
# libaccord_drop{2,3}.so, -DACCORD_BF16_DROP=k) vs the product build at c5.
set -x
L=$PWD/paper_2412_11554_b200
ACCORD_LIB=$L/libaccord_drop3.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "f32_small or config2 or dense_candidate or degenerate" > gpurun_out/pytest_gpu45_drop3.log 2>&1; echo pt=$?
for i in 1 2; do
for v in base drop2 drop3; do
  if [ $v = base ]; then lib=$L/libaccord.so; else lib=$L/libaccord_$v.so; fi
  ACCORD_LIB=$lib timeout 600 python bench.py --config 5 --no-e2e --no-cpu-baseline > gpurun_out/b45_c5_${v}_$i.json 2>gpurun_out/b45_c5_${v}_$i.log
done
done
tail -2 gpurun_out/pytest_gpu45_drop3.log
