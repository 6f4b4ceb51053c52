# Round 2, third GPU call: workspace tests (destroy fix), refine variants
# (block / flat / TMA ring) for parity and speed (c3, c4, c5), ncu of the new refine.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_workspace.py -q --durations=5 > gpurun_out/r02c_ws.log 2>&1; echo ws=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x > gpurun_out/r02c_parity_tma.log 2>&1; echo par_tma=$?
ACCORD_REFINE=flat timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x > gpurun_out/r02c_parity_flat.log 2>&1; echo par_flat=$?
for c in 3 4 5; do for k in block flat tma; do
  ACCORD_REFINE=$k timeout 900 python bench.py --config $c --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02c_bench_c${c}_$k.json 2> gpurun_out/r02c_bench_c${c}_$k.log; echo b$c$k=$?
done; done
timeout 1200 ncu --set full --import-source on --clock-control none -k 'regex:refine' -s 2 -c 2 \
  -o gpurun_out/r02c_refine_c5 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02c_ncu_refine.log 2>&1; echo ncu=$?
