#!/bin/bash
for v in -1 12 14 17 18 9; do
  echo "variant $v"
  TDVP_RJ_VARIANT=$v timeout 300 python tools/lanes_bench.py c2sat 1 8 2>&1 | tail -2
done
