#!/bin/bash
timeout 300 python tools/lanes_bench.py c2sat 8 2>&1 | tail -2
TDVP_LZ_FUSED=0 timeout 300 python tools/lanes_bench.py c2sat 8 2>&1 | tail -2
TDVP_LZ_FUSED=0 timeout 300 python tools/lanes_bench.py c2sat 1 2>&1 | tail -2
timeout 300 python tools/lanes_bench.py c2sat 16 2>&1 | tail -2
nproc
