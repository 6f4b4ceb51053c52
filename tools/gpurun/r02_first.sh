# Round 2, first GPU call: the new filter-audit / lambda_max / full-size tests,
# then the whole GPU suite, smoke, and the c5 bench line.
set -x
mkdir -p gpurun_out
rm -f gpurun_out/filter_audit.jsonl
timeout 1500 python -m pytest tests/test_gpu_filter.py -q -x --durations=10 > gpurun_out/r02a_filter.log 2>&1; echo filter=$?
timeout 2400 python -m pytest tests -m gpu -q --durations=12 --ignore=tests/test_gpu_filter.py > gpurun_out/r02a_pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/r02a_bench_c5.json 2> gpurun_out/r02a_bench_c5.log; echo b5=$?
