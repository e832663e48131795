#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "syev or eig or tridiag" > gpurun_out/eig_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/eig_tests.log
run() { echo "== $*"; env "$@" timeout 300 python scripts/eig_bench.py 120 200 300 400 500 600 1000 2>&1 | grep -v Warn; }
run GCG_TRIMODE=c > gpurun_out/eig_ab.log
run GCG_TRIMODE=g >> gpurun_out/eig_ab.log
run GCG_TRIMODE=o >> gpurun_out/eig_ab.log
cat gpurun_out/eig_ab.log
