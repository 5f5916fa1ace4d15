#!/bin/bash
python -m paper_1912_06127_b200.build > /tmp/build.log 2>&1 || { cat /tmp/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "svd" 2>&1 | tail -2
timeout 300 python tools/dbg_svd.py 2>&1 | grep -E "^1 |^2 "
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "config5 and 1" 2>&1 | grep -E "Error|assert|^E |passed|failed" | head -20
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1
