#!/usr/bin/env bash
set -u
run() { echo "== $*"; env "$@" timeout 600 python scripts/cg_bench.py ${CFGS:-2 3 4} 2>&1 | grep sweeps; }
for i in 1 2; do
run GCG_PDL=0
run GCG_PDL=1
done
for v in 0 1; do
GCG_PDL=$v timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pdl$v.log 2>&1; echo "bench pdl=$v rc=$?"; tail -1 gpurun_out/bench_pdl$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['iterations'], d['roofline']['frac'])"
done
