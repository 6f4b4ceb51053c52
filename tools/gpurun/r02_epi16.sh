# Epilogue width A-B, same box: int8 GEMM with 8 (default) vs 16 epilogue
# warps at c5; bf16 GEMM with 4 (default) vs 8 (bf16 throughout, AUTO off).
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_i8.py -k "config2_every_iteration or ragged" > gpurun_out/e16_pytest.log 2>&1; echo pt=$?
ACCORD_GEMM_VARIANT=4 timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_i8.py -k "config2_every_iteration or ragged or matches_bf16" > gpurun_out/e16_pytest_v4.log 2>&1; echo pt4=$?
for rep in 1 2; do for v in 0 4; do
  ACCORD_GEMM_VARIANT=$v timeout 900 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/e16_i8_v${v}_$rep.json 2> gpurun_out/e16_i8_v${v}_$rep.log; echo i8v$v$rep=$?
done; done
for v in 0 3; do
  ACCORD_AUTO_GEMM=bf16 ACCORD_GEMM_VARIANT=$v timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/e16_bf16_v$v.json 2> gpurun_out/e16_bf16_v$v.log; echo bfv$v=$?
done
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_workspace.py > gpurun_out/e16_pytest_ws.log 2>&1; echo ws=$?
