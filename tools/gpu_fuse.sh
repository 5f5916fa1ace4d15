#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_diagnostics.py -q -x > gpurun_out/fu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fu.log
for f in 0 1; do echo "FUSE=$f"; TDVP_HEFF_FUSE=$f timeout 300 python microbench.py --heff --chis 64,128,256,512 > gpurun_out/fh.log 2>&1; grep '"D": 5' gpurun_out/fh.log; done
for f in 0 1; do TDVP_HEFF_FUSE=$f LB_TIMING=1 timeout 300 python tools/lanes_bench.py c2sat 1 2>&1 | tail -2; done
