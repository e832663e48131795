#!/usr/bin/env bash
set -u
for V in "GCG_X=0" "GCG_PDL=0" "GCG_CG_PREFETCH=0" "GCG_PDL=0 GCG_CG_PREFETCH=0"; do
  echo "== $V: $(env $V timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],4), d['roofline']['frac'], {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items()})")"
done
for V in "GCG_X=0" "GCG_SPMM_PANEL=0" "GCG_SPMM_PANEL=0 GCG_CG_PREFETCH=0" "GCG_SPMM_PANEL=0 GCG_PDL=0"; do
  echo "== cfg4 $V: $(env $V timeout 300 python scripts/cg_bench.py 4 2>&1 | grep sweeps)"
done
