#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for v in 0 1 0 1; do
GCG_PDL=$v timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pdl$v.log 2>&1; echo "bench pdl=$v rc=$?"; tail -1 gpurun_out/bench_pdl$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['iterations'], d['roofline']['frac'])"
done
python scripts/prof_gaps.py > gpurun_out/gaps.txt 2>&1; head -12 gpurun_out/gaps.txt
