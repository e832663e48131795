#!/usr/bin/env bash
set -u
run() { echo "== $*"; env "$@" timeout 600 python scripts/cg_bench.py ${CFGS:-2 3 4} 2>&1 | grep sweeps; }
run GCG_X=0
run GCG_CG_STAGES=0
run GCG_CG_STAGES=1
run GCG_CG_STAGES=2
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -q -x -k "cg or spmm" > gpurun_out/cg_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/cg_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ab3.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_ab3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], json.dumps(d['kernels']))"
