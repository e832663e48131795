#!/usr/bin/env bash
# cfg4 / cfg5 SpMM: row order (grid-stride vs contiguous CTA ranges) x column panel width,
# then ncu of the default cfg4 CG-form SpMM
set -u
mkdir -p gpurun_out
for O in 0 1; do for P in 0 20 40 52; do
  echo "== ORDER=$O PANEL=$P"
  GCG_SPMM_ORDER=$O GCG_SPMM_PANEL=$P timeout 300 python scripts/kbench_big.py 4 2>&1 | grep spmm
done; done > gpurun_out/spmm4_probe.log
cat gpurun_out/spmm4_probe.log
for O in 0 1; do for P in 0 32 64; do
  echo "== cfg5 ORDER=$O PANEL=$P"
  GCG_SPMM_ORDER=$O GCG_SPMM_PANEL=$P timeout 300 python scripts/kbench_big.py 5 2>&1 | grep spmm
done; done > gpurun_out/spmm5_probe.log
cat gpurun_out/spmm5_probe.log
ncu --set full --clock-control none -k regex:spmm_csr_kernel -s 3 -c 1 -o gpurun_out/full_spmm4 \
    python scripts/kbench_big.py 4 > gpurun_out/ncu_spmm4.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py gpurun_out/full_spmm4.ncu-rep > gpurun_out/ncu_sum_spmm4.txt 2>&1; head -32 gpurun_out/ncu_sum_spmm4.txt
