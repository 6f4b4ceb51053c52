set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 -k "not fullsize" > gpurun_out/pytest_gpu2.log 2>&1; echo pytest=$?
timeout 600 python tools/gemm_sweep.py 5 64,0 32,0 16,0 24,0 > gpurun_out/sweep.log 2>&1; echo sweep=$?
timeout 900 python bench.py > gpurun_out/bench_c5_v6.json 2> gpurun_out/bench_c5_v6.log; echo bench=$?
tail -3 gpurun_out/pytest_gpu2.log
