#!/usr/bin/env bash
# ncu --set full of the k=20 CG-form SpMM launch in kbench (after a plain run exits 0)
set -u
mkdir -p gpurun_out
CMD="python scripts/kbench.py 2"
$CMD > gpurun_out/kb_plain.log 2>&1 || { echo plain failed; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:spmm_csr -s ${SKIP:-75} -c 1 \
    -o gpurun_out/${OUT:-kb_spmm} $CMD > gpurun_out/ncu_spmm.log 2>&1; echo "spmm rc=$?"
