#!/usr/bin/env bash
# one ncu --set full capture of the fused CG sweep inside cg_bench (cfg2), raw page kept
set -u
mkdir -p gpurun_out
CFG=${CFG:-2}
timeout 300 python scripts/cg_bench.py $CFG > gpurun_out/cgb.log 2>&1 || { tail gpurun_out/cgb.log; exit 1; }
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:spmm_csr_kernel" -s ${SKIP:-40} -c 1 \
    -o gpurun_out/full_sweep_raw python scripts/cg_bench.py $CFG > gpurun_out/ncu_sweep_raw.log 2>&1
echo "rc=$?"
ncu -i gpurun_out/full_sweep_raw.ncu-rep --page raw --csv > gpurun_out/sweep_raw.csv 2>&1
ncu -i gpurun_out/full_sweep_raw.ncu-rep --page details > gpurun_out/sweep_details.txt 2>&1
