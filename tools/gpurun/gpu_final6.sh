# Round-end measurement set after the symmetric first GEMM (one B200): all GPU tests, smoke, parity report
# (configs 1-6), bench lines c3-c6, reference arm, GEMM ncu (steady state),
# launch list of the timed c5 steps.
set -x
timeout 2700 python -m pytest tests -m gpu -q --durations=6 > gpurun_out/final6_pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final6_smoke.log 2>&1; echo smoke=$?
timeout 1800 python tools/parity_report.py > gpurun_out/final6_parity_report.json 2> gpurun_out/final6_parity_report.log; echo parity=$?
timeout 900 python bench.py > gpurun_out/final6_bench_c5.json 2> gpurun_out/final6_bench_c5.log; echo b5=$?
for c in 4 3 6; do timeout 900 python bench.py --config $c > gpurun_out/final6_bench_c$c.json 2> gpurun_out/final6_bench_c$c.log; echo b$c=$?; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final6_ref.json 2> gpurun_out/final6_ref.log; echo ref=$?
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final6_plain.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^(?!.*pi_)' -c 400 --csv --log-file gpurun_out/final6_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final6_ncu_launches.log 2>&1; echo launches=$?
timeout 600 python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/final6_plain2.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 5 -c 1 -o gpurun_out/final6_prof_gemm_c5 python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/final6_ncu_gemm.log 2>&1; echo ncu=$?
