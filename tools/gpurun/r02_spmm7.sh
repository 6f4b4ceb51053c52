# Round 2, fifth session: (1) gather microbenchmark with prefetched indices
# (bulk ring one-lane / all-lane issue, LDGSTS ring; float-sum and paired-f64
# consumers), (2) SpMM parity tests on the nested-loop consumer, (3) same-box
# A-B head library vs nested-loop consumer, ring stages 8 / 16.
set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/gather_bench.cu -o /tmp/gather_bench && \
  timeout 300 /tmp/gather_bench > gpurun_out/s7_gather_bench.txt 2>&1; echo gather=$?
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "spmm or bitwise or paired or f32_small or config2 or dense" > gpurun_out/s7_pytest.log 2>&1; echo pt=$?
for rep in 1 2; do
for v in head nest nest16; do
  case $v in head) E="ACCORD_LIB=$PWD/paper_2412_11554_b200/libaccord_head.so";; nest) E="ACCORD_SPMM_STAGES=8";; nest16) E="ACCORD_SPMM_STAGES=16";; esac
  env $E ACCORD_TRACE=1 timeout 900 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/s7_${v}_$rep.json 2> gpurun_out/s7_${v}_$rep.log; echo $v$rep=$?
done; done
