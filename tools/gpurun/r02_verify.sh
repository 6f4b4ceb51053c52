# Verification of the current build: GPU suite, smoke, c5 bench line.
set -x
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/ver_pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ver_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/ver_bench_c5.json 2> gpurun_out/ver_bench_c5.log; echo b5=$?
