#!/bin/bash
# after the pool-chunk fix (>= 2048 entries: a mirrored emission batch fits)
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k symmetric > gpurun_out/pytest_gpu49_sym.log 2>&1; echo sym=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu49.log 2>&1; echo pt=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke49.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/b49_c5.json 2> gpurun_out/b49_c5.log
tail -2 gpurun_out/pytest_gpu49.log
