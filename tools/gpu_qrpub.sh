#!/bin/bash
for v in 1 2 8; do
  echo "QR_PUB=$v"; TDVP_LIB=$PWD/qrpub_tmp/libtdvp_$v.so timeout 300 python microbench.py --svd --svd-n 256,512 --reps 5 --svd-kind halfsmall 2>&1 | tail -2
done
echo "QR_PUB=4"; timeout 300 python microbench.py --svd --svd-n 256,512 --reps 5 --svd-kind halfsmall 2>&1 | tail -2
