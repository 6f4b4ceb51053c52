set -x
timeout 2400 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu6.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/bench_c5_v7.json 2> gpurun_out/bench_c5_v7.log; echo bench=$?
timeout 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/prof_gemm_c5_v7 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu7.log 2>&1; echo ncu=$?
tail -3 gpurun_out/pytest_gpu6.log
