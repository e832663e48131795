#!/usr/bin/env bash
CMD="python scripts/time_cfg.py 2 6"
$CMD > gpurun_out/plain_t6.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_t6.csv $CMD > gpurun_out/ncu_t6.log 2>&1
echo rc=$?
cat gpurun_out/plain_t6.log
