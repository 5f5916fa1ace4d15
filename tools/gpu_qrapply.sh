#!/bin/bash
for nt in 256 128 64; do echo "APPLY_NT=$nt"; TDVP_QR_APPLY_NT=$nt timeout 300 python microbench.py --svd --svd-n 128,256 --reps 10 --svd-kind halfsmall 2>&1 | tail -2; done
TDVP_QR_APPLY_NT=64 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k svd > gpurun_out/qa.log 2>&1; tail -1 gpurun_out/qa.log
TDVP_QR_APPLY_NT=128 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k svd > gpurun_out/qa.log 2>&1; tail -1 gpurun_out/qa.log
