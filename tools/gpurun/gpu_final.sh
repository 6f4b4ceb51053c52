# Round-end measurement set (one B200): tests, parity report, bench lines,
# GEMM ncu capture (traffic), launch list of the timed steps.
set -x
timeout 2400 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/final_pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke=$?
timeout 1500 python tools/parity_report.py > gpurun_out/final_parity_report.json 2> gpurun_out/final_parity_report.log; echo parity=$?
timeout 900 python bench.py > gpurun_out/final_bench_c5.json 2> gpurun_out/final_bench_c5.log; echo b5=$?
timeout 900 python bench.py --config 4 > gpurun_out/final_bench_c4.json 2> gpurun_out/final_bench_c4.log; echo b4=$?
timeout 900 python bench.py --config 3 > gpurun_out/final_bench_c3.json 2> gpurun_out/final_bench_c3.log; echo b3=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.log; echo ref=$?
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final_plain.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^(?!.*pi_)' -c 400 --csv --log-file gpurun_out/final_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final_ncu_launches.log 2>&1; echo launches=$?
timeout 600 python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/final_plain2.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 5 -c 1 -o gpurun_out/final_prof_gemm_c5 python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/final_ncu_gemm.log 2>&1; echo ncu=$?
