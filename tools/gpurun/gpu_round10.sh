set -x
timeout 900 python -m pytest tests/test_multirank.py -m gpu -x -q > gpurun_out/pytest_gpu10.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain10.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^(?!.*pi_)' -c 400 --csv --log-file gpurun_out/launches_c5_v10.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu10.log 2>&1; echo ncu=$?
tail -3 gpurun_out/pytest_gpu10.log
