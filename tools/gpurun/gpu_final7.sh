# Round-end set on the final build (symmetric first GEMM + line search from
# Omega = I): all GPU tests, smoke, parity report c1-c6, bench lines c5/c4/c3/c6.
set -x
timeout 2700 python -m pytest tests -m gpu -q --durations=6 > gpurun_out/final7_pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final7_smoke.log 2>&1; echo smoke=$?
timeout 1800 python tools/parity_report.py > gpurun_out/final7_parity_report.json 2> gpurun_out/final7_parity_report.log; echo parity=$?
timeout 900 python bench.py > gpurun_out/final7_bench_c5.json 2> gpurun_out/final7_bench_c5.log; echo b5=$?
for c in 4 3 6; do timeout 900 python bench.py --config $c > gpurun_out/final7_bench_c$c.json 2> gpurun_out/final7_bench_c$c.log; echo b$c=$?; done
