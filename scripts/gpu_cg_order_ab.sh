#!/usr/bin/env bash
# contiguous row ranges per CTA (y +- 1 neighbours L1-resident) x staged own-row streams
set -u
run() { echo "== $*"; env "$@" timeout 600 python scripts/cg_bench.py ${CFGS:-2 4} 2>&1 | grep sweeps; }
run GCG_CG_STAGES=0 GCG_SPMM_ORDER=0
run GCG_CG_STAGES=0 GCG_SPMM_ORDER=1
run GCG_CG_STAGES=1 GCG_SPMM_ORDER=1
run GCG_CG_STAGES=2 GCG_SPMM_ORDER=1
run GCG_CG_STAGES=0 GCG_SPMM_ORDER=1 GCG_CG_PREFETCH=0
