#!/bin/bash
# e2e amortisation: K = 20 iterations from scratch (c5)
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b55_c5_k20.json 2> gpurun_out/b55_c5_k20.log
