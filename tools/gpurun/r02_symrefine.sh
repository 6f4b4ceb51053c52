# Symmetric refine at Omega = I (entries k >= i gathered, the rest copied from
# their twins): parity tests, then c5 A-B against ACCORD_REFINE_NOSYM=1.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "symmetric or first_iteration or bitwise" > gpurun_out/symref_pytest.log 2>&1; echo pt=$?
timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_fullsize.py -k config3_full_oracle > gpurun_out/symref_c3.log 2>&1; echo pc=$?
for rep in 1 2; do for k in 0 1; do
  if [ $k = 1 ]; then export ACCORD_REFINE_NOSYM=1; else unset ACCORD_REFINE_NOSYM; fi
  timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/symref_c5_${k}_$rep.json 2> gpurun_out/symref_c5_${k}_$rep.log; echo b$k$rep=$?
done; done
