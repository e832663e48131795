#!/usr/bin/env bash
# launch list (durations) of one cuSOLVER syevd at m = 200 (after a plain run exits 0)
set -u
mkdir -p gpurun_out
python scripts/syev_ab.py > gpurun_out/syev_plain.log 2>&1 || { echo plain failed; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/syev_launches.csv \
    python scripts/syev_ab.py > gpurun_out/ncu_syev.log 2>&1; echo "ncu rc=$?"
