#!/bin/bash
python -m paper_1912_06127_b200.build > /tmp/build.log 2>&1 || { cat /tmp/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "svd" 2>&1 | tail -2
timeout 300 python tools/dbg_svd.py 2>&1 | grep -v "e-1[3456] UU" | tail -25
for v in 11 6 10 9; do
  for k in halfsmall graded gauss; do
    echo "v$v $k $(TDVP_RJ_VARIANT=$v timeout 120 python microbench.py --svd --svd-n 256 --svd-kind $k 2>&1 | grep kernel)"
  done
done
for v in 7 8; do echo "v$v n512 $(TDVP_RJ_VARIANT=$v timeout 120 python microbench.py --svd --svd-n 512 --svd-kind halfsmall 2>&1 | grep kernel)"; done
echo "n1024 $(timeout 200 python microbench.py --svd --svd-n 1024 --svd-kind halfsmall 2>&1 | grep kernel)"
