# Round 2, sixth GPU call: fused Lanczos pass (create time), refine 128 threads,
# full-oracle c3 golden, filter + L tests, compute-sanitizer on the kernels.
set -x
mkdir -p gpurun_out
ACCORD_TRACE=1 timeout 900 python tools/create_timing.py 5 > gpurun_out/r02f_create.log 2>&1; echo create=$?
ACCORD_GRAM_2PASS=1 ACCORD_TRACE=1 timeout 900 python tools/create_timing.py 5 > gpurun_out/r02f_create_2pass.log 2>&1; echo create2=$?
timeout 1800 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "config3_full or lanczos or identity or beyond or tma_spmm" --durations=8 > gpurun_out/r02f_tests.log 2>&1; echo tests=$?
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/r02f_bench_c5.json 2> gpurun_out/r02f_bench_c5.log; echo b5=$?
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_bench_c3.json 2> gpurun_out/r02f_bench_c3.log; echo b3=$?
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/r02f_sanitize_$tool.log 2>&1; echo $tool=$?
done
