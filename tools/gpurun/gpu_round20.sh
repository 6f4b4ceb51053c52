set -x
ACCORD_TRACE=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b20.json 2> gpurun_out/b20_trace.log; echo b=$?
