#!/usr/bin/env bash
set -u
run() { echo "== $*"; env "$@" timeout 300 python scripts/cg_bench.py 2 4 2>&1 | grep sweeps; }
run GCG_X=0
run GCG_CG_MINB=4
run GCG_SPMM_PANEL=0
run GCG_SPMM_PANEL=20
run GCG_SPMM_PANEL=52
run GCG_CG_PREFETCH=0
run GCG_PDL=0
