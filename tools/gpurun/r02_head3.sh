# Round 2, third session: re-verify the restored tree (all GPU tests incl.
# the workspace test after the 2 M-entry default pool, smoke, c5 bench line).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/h3_pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h3_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/h3_bench_c5.json 2> gpurun_out/h3_bench_c5.log; echo b5=$?
