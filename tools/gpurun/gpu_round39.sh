timeout 1200 python -m pytest tests/test_multirank.py -m gpu -x -q -k "config5" > gpurun_out/pytest_gpu39.log 2>&1; echo pt=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke39.log 2>&1; echo smoke=$?
tail -2 gpurun_out/pytest_gpu39.log; tail -1 gpurun_out/smoke39.log
