set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -m gpu -x -q -k "not dense_candidate" > gpurun_out/pytest_gpu7.log 2>&1; echo pytest=$?
timeout 600 python tools/gemm_sweep.py 5 0,32,0,0 0,32,0,1 0,64,0,1 0,32,0,2 > gpurun_out/sweep7.log 2>&1; echo sweep=$?
for h in 0 1; do
  timeout 600 python tools/gemm_sweep.py 5 0,32,0,$h > gpurun_out/sweep7_h$h.log 2>&1 && \
  timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:gemm_tc -s 3 -c 1 --csv --log-file gpurun_out/ncu7_dram_h$h.csv python tools/gemm_sweep.py 5 0,32,0,$h > gpurun_out/ncu7_h$h.log 2>&1; echo ncu$h=$?
done
tail -3 gpurun_out/pytest_gpu7.log
