#!/usr/bin/env bash
set -u
timeout 900 python -m pytest tests/test_gpu_orth.py tests/test_gpu_solver.py tests/test_gpu_parity.py -q -x --timeout 300 2>&1 | tail -2
for i in 1 2; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_q.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['iterations'])"
done
