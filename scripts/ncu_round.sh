#!/usr/bin/env bash
# plain run, then ncu launch list + full captures of the top kernels (1 GPU)
set -u
CMD="python scripts/time_cfg.py 2 3"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
for K in spmm_csr_kernel gram_kernel lincomb_kernel cg_update_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 40 -c 2 -o gpurun_out/prof_$K $CMD > gpurun_out/ncu_$K.log 2>&1
  echo "$K rc=$?"
done
ls -la gpurun_out
