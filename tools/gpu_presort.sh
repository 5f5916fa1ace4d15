#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_diagnostics.py -q -x 2>&1 | tail -3
timeout 300 python tools/lanes_bench.py c2sat 1 8 2>&1 | tail -2
TDVP_SVD_PRESORT=0 timeout 300 python tools/lanes_bench.py c2sat 1 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_configs.py -q -x 2>&1 | tail -3
