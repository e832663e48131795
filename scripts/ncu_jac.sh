#!/usr/bin/env bash
CMD="python scripts/kbench.py 2"
$CMD > gpurun_out/kb_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:syev_jacobi -s 2 -c 1 -o gpurun_out/kb_jac $CMD > gpurun_out/ncu_jac.log 2>&1; echo "rc=$?"
