#!/usr/bin/env bash
# A/B of the staged CG sweep (bulk-copied p/q/x ring per warp) against the prefetching one
set -u
mkdir -p gpurun_out
run() { echo "== $*"; env "$@" timeout 600 python scripts/cg_bench.py ${CFGS:-2 4} 2>&1 | grep sweeps; }
run GCG_CG_STAGES=0
run GCG_CG_STAGES=1
run GCG_CG_STAGES=2
run GCG_CG_STAGES=3
run GCG_CG_STAGES=4
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -q -x -k "cg" > gpurun_out/cg_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/cg_tests.log
for st in 0 2; do
GCG_CG_STAGES=$st timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_st$st.log 2>&1; echo "bench stages=$st rc=$?"; tail -1 gpurun_out/bench_st$st.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], json.dumps(d['kernels']))"
done
