#!/usr/bin/env bash
set -u
run() { echo "== $*"; env "$@" timeout 600 python scripts/cg_bench.py ${CFGS:-2 3 4} 2>&1 | grep -E "sweeps"; }
for i in 1 2; do
run GCG_CG_UPD_ORDER=0
run GCG_CG_UPD_ORDER=1
run GCG_CG_UPD_ORDER=2
done
