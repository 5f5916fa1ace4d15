#!/bin/bash
# Round-1 final profiling: bench (plain), ncu full capture of the dominant kernel
# (rjac2 Jacobi) and of the QR kernel inside the bench step, launch list of part of a step.
mkdir -p gpurun_out
python -m paper_1912_06127_b200.build > /dev/null 2>&1
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/p_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rjac2 -s 40 -c 1 -o gpurun_out/bench_rjac2 \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/p_ncu1.log 2>&1
echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"qrc3|qr_apply|zgemm|chanmix|lz_pass" -s 2000 -c 12 -o gpurun_out/bench_misc \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/p_ncu2.log 2>&1
echo "ncu2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 16000 -c 4000 --csv --log-file gpurun_out/launches_r1.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/p_ncu3.log 2>&1
echo "ncu3 rc=$?"
ls -la gpurun_out | tail -8
