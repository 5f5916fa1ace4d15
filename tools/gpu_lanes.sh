#!/bin/bash
# segment lanes: parity tests + timing (1 GPU)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_diagnostics.py -q -x -k "segmented or infidelity or long_range or reorth" 2>&1 | tail -5
timeout 600 python tools/lanes_bench.py c2sat 1 2 4 8 2>&1 | tail -8
TDVP_LANES=0 timeout 600 python tools/lanes_bench.py c2sat 2 8 2>&1 | tail -4
