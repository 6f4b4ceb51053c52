# Round 2, 11th GPU call: where the c3 / c4 from-scratch time goes (create
# phases + first-iteration trace).
set -x
mkdir -p gpurun_out
ACCORD_TRACE=1 timeout 600 python tools/create_timing.py 3 > gpurun_out/r02k_create_c3.log 2>&1; echo cr3=$?
ACCORD_TRACE=1 timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02k_bench_c3.json 2> gpurun_out/r02k_bench_c3.log; echo b3=$?
ACCORD_TRACE=1 timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02k_bench_c4.json 2> gpurun_out/r02k_bench_c4.log; echo b4=$?
