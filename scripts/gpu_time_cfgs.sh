#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
for C in 1 3 4; do
  timeout 900 python scripts/time_cfg.py $C > gpurun_out/time_cfg$C.txt 2>&1; echo "cfg$C rc=$?"; tail -4 gpurun_out/time_cfg$C.txt
done
