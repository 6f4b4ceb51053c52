# Round 2c: __syncwarp before the finalize reductions (c6 regression): SpMM
# parity / bitwise tests, smoke, c6 and c5 bench lines against the previous
# commit's numbers.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "spmm or bitwise or paired or f32_small or config2 or dense" > gpurun_out/c6fix_pytest.log 2>&1; echo pt=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c6fix_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py --config 6 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c6fix_c6.json 2> gpurun_out/c6fix_c6.log; echo c6=$?
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c6fix_c4.json 2> gpurun_out/c6fix_c4.log; echo c4=$?
timeout 900 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c6fix_c5.json 2> gpurun_out/c6fix_c5.log; echo c5=$?
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_fullsize.py > gpurun_out/c6fix_pytest_fullsize.log 2>&1; echo ptf=$?
