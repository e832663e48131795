#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
for M in c o g; do
  GCG_TRIMODE=$M timeout 300 python scripts/eig_bench.py 80 120 160 200 224 300 400 500 600 > gpurun_out/eig_mode_$M.log 2>&1; echo "mode $M rc=$?"; cat gpurun_out/eig_mode_$M.log
done
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "syev or eig or tridiag" > gpurun_out/eig_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/eig_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-400
