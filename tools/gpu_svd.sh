#!/bin/bash
# SVD iteration on the GPU box: parity tests, microbench, phase profile, smoke.
mkdir -p gpurun_out
python -m paper_1912_06127_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "svd" 2>&1 | tail -15
TDVP_SVD_PROF=1 timeout 300 python microbench.py --svd --svd-n 16,64,128,256,512,1024 2>&1 | tail -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1
