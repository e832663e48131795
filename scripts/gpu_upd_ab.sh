#!/usr/bin/env bash
# A/B: bulk-copy r-update (default) vs the register-streamed kernel
set -u
run() { echo "== $*"; env "$@" timeout 600 python scripts/cg_bench.py ${CFGS:-2 3 4} 2>&1 | grep sweeps; }
for i in 1 2; do
run GCG_CG_UPD_BULK=0
run GCG_CG_UPD_BULK=1
done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -q -x -k "cg or golden or cfg2" > gpurun_out/cg_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/cg_tests.log
for v in 0 1; do
GCG_CG_UPD_BULK=$v timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_upd$v.log 2>&1; echo "bench bulk=$v rc=$?"; tail -1 gpurun_out/bench_upd$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], json.dumps(d['kernels']))"
done
