#!/usr/bin/env bash
# A/B: Gram stages as one ascending window (GCG_GRAM_INTER) + LinComb tiles descending (GCG_LC_DESC)
set -u
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_orth.py -q -x --timeout 300 2>&1 | tail -2
for v in "0 0" "1 1" "1 0" "0 1" "0 0" "1 1"; do
set -- $v
GCG_GRAM_INTER=$1 GCG_LC_DESC=$2 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pp.log 2>&1; echo "bench inter=$1 desc=$2 rc=$?"; tail -1 gpurun_out/bench_pp.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['iterations'], {k:round(v['ms_per_step'],1) for k,v in d['kernels'].items()})"
done
