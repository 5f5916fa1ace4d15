#!/bin/bash
# SVD variant sweep + phase profile on the GPU box
python -m paper_1912_06127_b200.build > /tmp/build.log 2>&1 || { cat /tmp/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "svd" 2>&1 | tail -3
for v in 0 1 5 99; do
  echo "== variant $v"
  TDVP_RJ_VARIANT=$v TDVP_SVD_PROF=2 timeout 120 python microbench.py --svd --svd-n 256 2>&1 | grep -E "rjac|svd" | awk 'NR%5==1 || /kernel/'
done
for v in 2 3 4; do
  echo "== variant $v"
  TDVP_RJ_VARIANT=$v TDVP_SVD_PROF=2 timeout 120 python microbench.py --svd --svd-n 512 2>&1 | grep -E "rjac|svd" | awk 'NR%5==1 || /kernel/'
done
timeout 300 python tools/dbg_svd.py 2>&1 | tail -40
