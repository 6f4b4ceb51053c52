set -x
timeout 1500 python tools/parity_report.py > gpurun_out/parity_report.json 2> gpurun_out/parity_report.log; echo parity=$?
timeout 900 python bench.py --config 5 > gpurun_out/bench_c5_v8.json 2> gpurun_out/bench_c5_v8.log; echo bench5=$?
timeout 900 python bench.py --config 4 > gpurun_out/bench_c4_v8.json 2> gpurun_out/bench_c4_v8.log; echo bench4=$?
timeout 900 python bench.py --config 3 > gpurun_out/bench_c3_v8.json 2> gpurun_out/bench_c3_v8.log; echo bench3=$?
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain8.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5_v8.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu8.log 2>&1; echo ncu=$?
