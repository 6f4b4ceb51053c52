#!/bin/bash
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py tests/test_multirank.py -m gpu -q > gpurun_out/pytest_gpu51.log 2>&1; echo pt=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke51.log 2>&1; echo smoke=$?
tail -3 gpurun_out/pytest_gpu51.log
