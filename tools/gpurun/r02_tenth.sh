# Round 2, tenth GPU call: supp Omega merged in the finalize (epilogue tests
# |acc| only) -- full GPU suite; same-box A-B against the previous epilogue
# (libaccord_oldepi.so: same library, round-2 epilogue with the support walk);
# first-iteration traces; other configs.
set -x
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r02j_pytest_gpu.log 2>&1; echo pytest=$?
for rep in 1 2; do
  ACCORD_TRACE=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02j_bench_c5_new$rep.json 2> gpurun_out/r02j_bench_c5_new$rep.log; echo new$rep=$?
  ACCORD_TRACE=1 ACCORD_LIB=paper_2412_11554_b200/libaccord_oldepi.so timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02j_bench_c5_old$rep.json 2> gpurun_out/r02j_bench_c5_old$rep.log; echo old$rep=$?
done
for c in 3 4 6; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02j_bench_c$c.json 2> gpurun_out/r02j_bench_c$c.log; echo b$c=$?; done
