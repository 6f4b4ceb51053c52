# int8 filter, second run: its GPU tests; c5 with AUTO's adaptive bf16 -> int8
# switch (traced) against bf16 only, same box; then the whole GPU suite.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_i8.py > gpurun_out/i8b_pytest.log 2>&1; echo pt=$?
for g in auto bf16; do
  ACCORD_TRACE=1 ACCORD_AUTO_GEMM=$g timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/i8b_c5_$g.json 2> gpurun_out/i8b_c5_$g.log; echo b$g=$?
done
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/i8b_pytest_all.log 2>&1; echo all=$?
