#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "svd" 2>&1 | tail -1
TDVP_SVD_PROF=1 timeout 600 python microbench.py --svd --svd-n 2048 --reps 1 --svd-kind halfsmall 2>&1 | tail -2
timeout 600 python microbench.py --svd --svd-n 2048 --reps 2 --svd-kind graded 2>&1 | tail -1
TDVP_RJ_VARIANT=99 timeout 600 python microbench.py --svd --svd-n 1024 --reps 2 --svd-kind halfsmall 2>&1 | tail -1
