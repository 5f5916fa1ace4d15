#!/bin/bash
for pc in 2 0; do
  TDVP_SVD_PRECOND=$pc timeout 600 python microbench.py --svd --svd-n 2048 --reps 2 --svd-kind halfsmall 2>&1 | tail -1
done
TDVP_SVD_PRECOND=2 timeout 600 python microbench.py --svd --svd-n 1024,2048 --reps 2 --svd-kind graded 2>&1 | tail -2
