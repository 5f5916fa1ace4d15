#!/bin/bash
# Round-1 (second session) validation + profiling: GPU tests, bench, ncu launch
# list of a c2sat step, full captures of the Jacobi kernel and the other hot kernels.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r1b_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r1b_pytest.log
timeout 900 python bench.py > gpurun_out/r1b_bench.json 2> gpurun_out/r1b_bench.err; echo "bench rc=$?"
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --lane-segments 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rjac2 -s 40 -c 1 -o gpurun_out/r1b_rjac2 $B > gpurun_out/r1b_ncu1.log 2>&1
echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qrc3|qr_apply|zgemm|chanmix|lz_iter|lz_tridiag" -s 3000 -c 14 -o gpurun_out/r1b_misc $B > gpurun_out/r1b_ncu2.log 2>&1
echo "ncu2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 16000 -c 4000 --csv --log-file gpurun_out/r1b_launches.csv $B > gpurun_out/r1b_ncu3.log 2>&1
echo "ncu3 rc=$?"
ls -la gpurun_out | grep r1b
