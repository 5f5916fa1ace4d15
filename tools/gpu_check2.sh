#!/bin/bash
mkdir -p gpurun_out
python -m paper_1912_06127_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -k "lanczos or config5 or bench or heff" 2>&1 | tail -4
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench2.json 2>&1; tail -1 gpurun_out/bench2.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 17500 -c 17500 --csv --log-file gpurun_out/launches2.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch2.log 2>&1; echo "ncu rc=$?"
