#!/bin/bash
# full GPU validation + bench + lanes on c3sat
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 400 gpurun_out/bench.err
LB_TIMING=1 timeout 900 python tools/lanes_bench.py c3sat 8 2>&1 | tail -3
