#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
GCG_TRIGRID=1 timeout 300 python scripts/eig_bench.py 120 160 200 224 > gpurun_out/eig_grid_small.log 2>&1; echo "eig grid rc=$?"; cat gpurun_out/eig_grid_small.log
timeout 300 python scripts/eig_bench.py 120 160 200 224 > gpurun_out/eig_cta_small.log 2>&1; echo "eig cta rc=$?"; cat gpurun_out/eig_cta_small.log
timeout 600 python scripts/prof_trace.py 20 21 > gpurun_out/trace.log 2>&1; echo "trace rc=$?"; tail -25 gpurun_out/trace.log
SKIP=200 bash scripts/ncu_cg.sh; head -30 gpurun_out/ncu_sum_cg_sweep.txt; head -30 gpurun_out/ncu_sum_cg_update.txt
