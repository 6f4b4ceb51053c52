set -x
timeout 900 python tools/gemm_sweep.py 5 0,32 > gpurun_out/sweep18_new.log 2>&1; echo s1=$?
ACCORD_LIB=$PWD/paper_2412_11554_b200/libaccord_prev.so timeout 900 python tools/gemm_sweep.py 5 0,32 > gpurun_out/sweep18_prev.log 2>&1; echo s2=$?
timeout 900 python tools/gemm_sweep.py 5 0,32 > gpurun_out/sweep18_new_b.log 2>&1; echo s3=$?
timeout 600 python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/plain18.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 5 -c 1 -o gpurun_out/prof_gemm_c5_steady python bench.py --steps 1 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ncu18.log 2>&1; echo ncu=$?
