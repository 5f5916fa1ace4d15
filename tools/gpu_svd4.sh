#!/bin/bash
# QR-preconditioned / rjac2 SVD checks on the GPU box
python -m paper_1912_06127_b200.build > /tmp/build.log 2>&1 || { cat /tmp/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "svd" 2>&1 | tail -3
timeout 300 python tools/dbg_svd.py 2>&1 | grep -E "256x256|512x512|300x700|^1 5|^2 5"
for pc in 0 2; do
 for v in 5 6 9 10; do
  echo "== precond $pc variant $v"
  TDVP_SVD_PRECOND=$pc TDVP_RJ_VARIANT=$v TDVP_SVD_PROF=1 timeout 120 python microbench.py --svd --svd-n 256 --svd-kind halfsmall 2>&1 | grep -E "rjac|svd" | awk 'NR%5==1 || /kernel/'
 done
done
for v in 7 8 10; do
  echo "== precond 2 variant $v n=512"
  TDVP_RJ_VARIANT=$v TDVP_SVD_PROF=1 timeout 120 python microbench.py --svd --svd-n 512 2>&1 | grep -E "rjac|svd" | awk 'NR%3==1 || /kernel/'
done
echo "== n=1024"
TDVP_SVD_PROF=1 timeout 200 python microbench.py --svd --svd-n 1024 2>&1 | grep -E "rjac|svd" | awk 'NR%3==1 || /kernel/'
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "config5 and 1" 2>&1 | grep -E "Error|assert|^E " | head -20
