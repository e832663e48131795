#!/usr/bin/env bash
# one gpurun call: kernel tests + kbench (spmm section) + bench
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/pytest_kern.log 2>&1; echo "kern rc=$?"; tail -3 gpurun_out/pytest_kern.log
timeout 600 python scripts/kbench.py ${KB_CFGS:-2} > gpurun_out/kbench.log 2>&1; echo "kbench rc=$?"; grep -i "spmm\|block CG\|cg_" gpurun_out/kbench.log
timeout 900 python bench.py --steps 3 --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-400
