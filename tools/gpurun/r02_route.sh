# Round 2c: TMA SpMM only for ldk % 256 == 0 (c6 routes to the block-per-row
# kernel): all GPU tests, smoke, c6 / c5 / c4 bench lines.
set -x
mkdir -p gpurun_out
timeout 300 python bench.py --config 6 --no-cpu-baseline > gpurun_out/rt_bench_c6.json 2> gpurun_out/rt_bench_c6.log; echo c6=$?
timeout 600 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/rt_bench_c5.json 2> gpurun_out/rt_bench_c5.log; echo c5=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rt_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/rt_pytest_gpu.log 2>&1; echo pytest=$?
