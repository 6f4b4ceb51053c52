# First hardware run of the int8 certified filter (ACCORD_GEMM_I8_FILTER):
# its GPU tests, a library-GEMM probe of the int8 / fp8 / bf16 rates under the
# power cap, and a same-box c5 A-B of the default (bf16 filter) vs int8.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_i8.py -k "not config3" > gpurun_out/i8a_pytest.log 2>&1; echo pt=$?
timeout 300 python tools/int8_probe.py > gpurun_out/i8a_probe.jsonl 2> gpurun_out/i8a_probe.log; echo probe=$?
for rep in 1; do for g in i8 bf16; do
  ACCORD_AUTO_GEMM=$g timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/i8a_c5_${g}_$rep.json 2> gpurun_out/i8a_c5_${g}_$rep.log; echo b$g$rep=$?
done; done
