timeout 1200 python -m pytest tests/test_multirank.py -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu34.log 2>&1; echo pt=$?
tail -15 gpurun_out/pytest_gpu34.log
