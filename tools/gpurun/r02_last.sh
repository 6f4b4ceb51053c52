# Round 2c: last sanity run of the tree as committed (the syncwarp experiment
# reverted, library rebuilt from 36865cf's source): smoke, SpMM parity /
# bitwise tests, c5 bench line.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.log 2>&1; echo smoke=$?
timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "bitwise or paired" > gpurun_out/last_pytest.log 2>&1; echo pt=$?
timeout 600 python bench.py --steps 3 --warmup 5 --no-cpu-baseline > gpurun_out/last_bench_c5.json 2> gpurun_out/last_bench_c5.log; echo c5=$?
timeout 300 python bench.py --config 6 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/last_bench_c6.json 2> gpurun_out/last_bench_c6.log; echo c6=$?
