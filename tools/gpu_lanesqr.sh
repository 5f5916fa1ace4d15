#!/bin/bash
for c in 16 8; do echo "QR_C=$c"; TDVP_QR_C=$c timeout 300 python tools/lanes_bench.py c2sat 8 16 2>&1 | tail -2; done
