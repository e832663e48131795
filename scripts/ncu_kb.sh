#!/usr/bin/env bash
set -u
CMD="python scripts/kbench.py 2"
$CMD > gpurun_out/kb_plain.log 2>&1 || { echo plain failed; exit 1; }
# 4th spmm pattern: k=20 CG form (contiguous, dots) is after 3 shapes x 23 launches
ncu --set full --clock-control none --import-source on -k regex:spmm_csr -s 75 -c 1 -o gpurun_out/kb_spmm2 $CMD > gpurun_out/ncu_kb1.log 2>&1; echo "spmm rc=$?"
ncu --set full --clock-control none --import-source on -k regex:gram_dmma -s 3 -c 1 -o gpurun_out/kb_gram2 $CMD > gpurun_out/ncu_kb2.log 2>&1; echo "gram rc=$?"
ncu --set full --clock-control none --import-source on -k regex:lincomb_dmma -s 3 -c 1 -o gpurun_out/kb_lincomb2 $CMD > gpurun_out/ncu_kb3.log 2>&1; echo "lincomb rc=$?"
