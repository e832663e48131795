#!/usr/bin/env bash
set -u
CMD="python scripts/kbench.py 2"
$CMD > gpurun_out/kb_plain.log 2>&1 || { echo plain failed; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:spmm_tiled -s 3 -c 1 -o gpurun_out/kb_spmm $CMD > gpurun_out/ncu_kb1.log 2>&1; echo "spmm rc=$?"
ncu --set full --clock-control none --import-source on -k regex:gram2 -s 3 -c 1 -o gpurun_out/kb_gram $CMD > gpurun_out/ncu_kb2.log 2>&1; echo "gram rc=$?"
ncu --set full --clock-control none --import-source on -k regex:lincomb2 -s 3 -c 1 -o gpurun_out/kb_lincomb $CMD > gpurun_out/ncu_kb3.log 2>&1; echo "lincomb rc=$?"
ncu --set full --clock-control none --import-source on -k regex:cg_update -s 3 -c 1 -o gpurun_out/kb_cgupd $CMD > gpurun_out/ncu_kb4.log 2>&1; echo "cgupd rc=$?"
