#!/bin/bash
for v in 14 21 22 6; do echo "TVAR=$v"; TDVP_RJ_TVARIANT=$v timeout 300 python tools/lanes_bench.py c2sat 8 2>&1 | tail -1; done
for v in 21 22; do echo "serial VAR=$v"; TDVP_RJ_VARIANT=$v timeout 300 python tools/lanes_bench.py c2sat 1 2>&1 | tail -1; done
TDVP_RJ_VARIANT=22 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k svd > gpurun_out/tv.log 2>&1; tail -1 gpurun_out/tv.log
