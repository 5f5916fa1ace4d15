#!/bin/bash
python -m paper_1912_06127_b200.build > /tmp/build.log 2>&1 || { cat /tmp/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1
TDVP_SVD_WARM=0 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-200
timeout 1200 python -m pytest tests/test_gpu_configs.py -x -q -k "bench or config2" 2>&1 | tail -3
