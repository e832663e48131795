#!/usr/bin/env bash
# ncu --set full of the fused CG sweep SpMM and the r-update inside a short cfg2 bench.
set -u
mkdir -p gpurun_out
SHORT="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$SHORT > gpurun_out/bench_short.log 2>&1 || { echo "short bench failed"; tail gpurun_out/bench_short.log; exit 1; }
tag=${TAG:-cg}
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:spmm_csr_kernel<\\(int\\)4, \\(int\\)1, \\(bool\\)0, \\(int\\)[12]>" -s ${SKIP:-60} -c 1 \
    -o gpurun_out/full_${tag}_sweep $SHORT > gpurun_out/ncu_${tag}_sweep.log 2>&1
echo "sweep rc=$?"
python scripts/ncu_summary.py gpurun_out/full_${tag}_sweep.ncu-rep > gpurun_out/ncu_sum_${tag}_sweep.txt 2>&1
[ -n "${NOUPD:-}" ] || ncu --set full --clock-control none --import-source on -k regex:cg_update -s ${SKIP:-60} -c 1 \
    -o gpurun_out/full_${tag}_update $SHORT > gpurun_out/ncu_${tag}_update.log 2>&1
echo "update rc=$?"
python scripts/ncu_summary.py gpurun_out/full_${tag}_update.ncu-rep > gpurun_out/ncu_sum_${tag}_update.txt 2>&1
rm -f gpurun_out/full_${tag}_update.ncu-rep
