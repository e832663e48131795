#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:tridiag_multi -s 2 -c 1 -o gpurun_out/tri200 \
    python scripts/eig_bench.py 200 > gpurun_out/ncu_tri200.log 2>&1; echo "rc=$?"
ncu -i gpurun_out/tri200.ncu-rep --page source --csv --print-source sass > gpurun_out/tri200_sass.csv 2>&1
ncu -i gpurun_out/tri200.ncu-rep --page source --csv > gpurun_out/tri200_src.csv 2>&1
python scripts/ncu_summary.py gpurun_out/tri200.ncu-rep | head -30
ls -la gpurun_out/tri200*
