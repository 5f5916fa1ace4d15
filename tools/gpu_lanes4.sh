#!/bin/bash
LB_TIMING=1 timeout 300 python tools/lanes_bench.py c2sat 1 2 4 8 2>&1 | tail -8
LB_TIMING=1 TDVP_RJ_VARIANT=14 timeout 300 python tools/lanes_bench.py c2sat 8 2>&1 | tail -2
