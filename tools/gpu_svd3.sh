#!/bin/bash
python -m paper_1912_06127_b200.build > /tmp/build.log 2>&1 || { cat /tmp/build.log; exit 1; }
for f in 0 1; do
 for v in 0 1 5; do
  echo "== fast $f variant $v"
  TDVP_RJ_FAST=$f TDVP_RJ_VARIANT=$v TDVP_SVD_PROF=2 timeout 120 python microbench.py --svd --svd-n 256 2>&1 | grep -E "rjac|svd" | awk 'NR%5==1 || /kernel/'
 done
 TDVP_RJ_FAST=$f timeout 300 python tools/dbg_svd.py 2>&1 | grep -E "256x256|512x512"
done
