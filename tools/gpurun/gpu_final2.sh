# Round-end re-measurement after the filter / SpMM-threshold changes.
set -x
timeout 2400 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/final2_pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2_smoke.log 2>&1; echo smoke=$?
timeout 1500 python tools/parity_report.py > gpurun_out/final2_parity_report.json 2> gpurun_out/final2_parity_report.log; echo parity=$?
timeout 900 python bench.py > gpurun_out/final2_bench_c5.json 2> gpurun_out/final2_bench_c5.log; echo b5=$?
timeout 900 python bench.py --config 4 > gpurun_out/final2_bench_c4.json 2> gpurun_out/final2_bench_c4.log; echo b4=$?
timeout 900 python bench.py --config 3 > gpurun_out/final2_bench_c3.json 2> gpurun_out/final2_bench_c3.log; echo b3=$?
