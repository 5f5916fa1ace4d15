#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "svd" 2>&1 | tail -1
for nt in 256 512; do
  echo "NT=$nt"
  TDVP_QR_NT=$nt TDVP_QR_PROF=1 timeout 300 python microbench.py --svd --svd-n 256 --reps 1 --svd-kind halfsmall 2>&1 | grep -A17 "qrc3 m=256" | tail -3
  TDVP_QR_NT=$nt timeout 300 python microbench.py --svd --svd-n 256,512 --reps 5 --svd-kind halfsmall 2>&1 | tail -2
  TDVP_QR_NT=$nt timeout 300 python tools/lanes_bench.py c2sat 1 2>&1 | tail -1
done
