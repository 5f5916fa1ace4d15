#!/bin/bash
for c in 16 8 12; do
  echo "C=$c"
  TDVP_QR_C=$c TDVP_QR_PROF=1 timeout 300 python microbench.py --svd --svd-n 256 --reps 1 --svd-kind halfsmall 2>&1 | grep -B2 -A17 "qrc3 m=256" | grep "cta" | tail -2
  TDVP_QR_C=$c timeout 300 python microbench.py --svd --svd-n 256,512 --reps 5 --svd-kind halfsmall 2>&1 | tail -2
done
