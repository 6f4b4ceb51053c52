set -x
for st in 8 12 16 6; do
ACCORD_SPMM_STAGES=$st timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/b21_st$st.json 2>/dev/null; echo st$st=$?
done
