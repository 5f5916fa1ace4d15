#!/bin/bash
# Round-1 profiling on the GPU box: launch list of one bench step, full captures
# of the H_eff GEMM stages (chi=128 and chi=1024) and of the SVD kernel (n=256).
set -x
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python microbench.py --heff --chis 128,1024 --reps 2 > gpurun_out/plain_heff.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:zgemm_dmma -s 8 -c 4 -o gpurun_out/heff_prof \
    python microbench.py --heff --chis 128,1024 --reps 2 > gpurun_out/ncu_heff.log 2>&1
python microbench.py --svd --svd-n 256 > gpurun_out/plain_svd.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:svd_coop -c 1 -o gpurun_out/svd_prof2 \
    python microbench.py --svd --svd-n 256 > gpurun_out/ncu_svd.log 2>&1
ls -la gpurun_out
