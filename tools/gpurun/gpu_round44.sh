#!/bin/bash
# Full GPU suite + smoke after the per-device attribute change.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke44.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke44.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu44.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu44.log
