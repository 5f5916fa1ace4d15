#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_diagnostics.py -q -x > gpurun_out/kt.log 2>&1; tail -2 gpurun_out/kt.log
for kt in 0 1e-6; do LB_KTOL=$kt LB_TIMING=1 timeout 300 python tools/lanes_bench.py c2sat 1 8 2>&1 | tail -4; done
