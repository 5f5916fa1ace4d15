#!/bin/bash
for g in 32 64 96 148 296; do
  echo "G=$g"; TDVP_LZ_G=$g LB_TIMING=1 timeout 300 python tools/lanes_bench.py c2sat 1 2>&1 | tail -2
done
