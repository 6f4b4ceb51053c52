# Round 2, fourth GPU call: float-float refine (default) vs float64, parity
# (default + the new n > 4096 / mixed-block / workspace tests), ncu of the refine.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_workspace.py -q > gpurun_out/r02d_ws.log 2>&1; echo ws=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py tests/test_multirank.py -q -x -m gpu > gpurun_out/r02d_parity.log 2>&1; echo par=$?
for c in 3 4 5; do for k in block ff; do
  ACCORD_REFINE=$k timeout 900 python bench.py --config $c --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02d_bench_c${c}_$k.json 2> gpurun_out/r02d_bench_c${c}_$k.log; echo b$c$k=$?
done; done
timeout 1200 ncu --set full --import-source on --clock-control none -k 'regex:refine' -s 2 -c 2 \
  -o gpurun_out/r02d_refine_c5 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02d_ncu_refine.log 2>&1; echo ncu=$?
