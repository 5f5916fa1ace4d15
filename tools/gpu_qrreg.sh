#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "svd" 2>&1 | tail -1
for v in 0 1 2; do
  echo "TDVP_QR_REG=$v"
  TDVP_QR_REG=$v TDVP_QR_PROF=1 timeout 300 python microbench.py --svd --svd-n 256 --reps 1 --svd-kind halfsmall 2>&1 | grep "cta 15" | tail -1
  TDVP_QR_REG=$v timeout 300 python microbench.py --svd --svd-n 128,256 --reps 5 --svd-kind halfsmall 2>&1 | tail -2
done
