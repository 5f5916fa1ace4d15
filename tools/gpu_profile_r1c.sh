#!/bin/bash
# bench + ncu evidence, exported to CSV on the box (the .ncu-rep files are too big to bring back)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r1c_bench.json 2> gpurun_out/r1c_bench.err; echo "bench rc=$?"
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --lane-segments 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rjac2 -s 40 -c 1 -o /tmp/r1c_rjac2 $B > gpurun_out/r1c_ncu1.log 2>&1
echo "ncu1 rc=$?"
ncu -i /tmp/r1c_rjac2.ncu-rep --page raw --csv > gpurun_out/r1c_rjac2_raw.csv 2>/dev/null
ncu -i /tmp/r1c_rjac2.ncu-rep --page details --csv > gpurun_out/r1c_rjac2_details.csv 2>/dev/null
ncu -i /tmp/r1c_rjac2.ncu-rep --page source --csv > gpurun_out/r1c_rjac2_source.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:"qrc3|qr_apply|zgemm|chanmix|lz_iter|lz_tridiag" -s 3000 -c 14 -o /tmp/r1c_misc $B > gpurun_out/r1c_ncu2.log 2>&1
echo "ncu2 rc=$?"
ncu -i /tmp/r1c_misc.ncu-rep --page raw --csv > gpurun_out/r1c_misc_raw.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 16000 -c 2500 --csv --log-file gpurun_out/r1c_launches.csv $B > gpurun_out/r1c_ncu3.log 2>&1
echo "ncu3 rc=$?"
du -sh gpurun_out; ls -la gpurun_out | grep r1c
