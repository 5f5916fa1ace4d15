#!/bin/bash
# full GPU validation: build, smoke, all gpu tests, bench
mkdir -p gpurun_out
python -m paper_1912_06127_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -8
timeout 900 python bench.py --steps 3 --warmup 3 2>&1 | tail -1 | tee gpurun_out/bench_full.json
