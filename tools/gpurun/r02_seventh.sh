# Round 2, seventh GPU call: symmetric first GEMM across ranks (multi-context,
# host transport), reproducibility, full GPU suite, c5 bench (regression check).
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_multirank.py -q -x -m gpu -k "symmetric or invariance or mixed" --durations=6 > gpurun_out/r02g_sym2.log 2>&1; echo sym2=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "reproducible" > gpurun_out/r02g_repro.log 2>&1; echo repro=$?
timeout 3000 python -m pytest tests -m gpu -q --durations=12 > gpurun_out/r02g_pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02g_bench_c5.json 2> gpurun_out/r02g_bench_c5.log; echo b5=$?
