#!/usr/bin/env bash
set -u
timeout 300 python scripts/cg_bench.py 2 4 2>&1 | grep sweeps
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -q -x > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t.log
timeout 900 python scripts/time_cfg.py 4 > gpurun_out/time_cfg4.txt 2>&1; tail -4 gpurun_out/time_cfg4.txt
timeout 900 python scripts/time_cfg.py 3 > gpurun_out/time_cfg3.txt 2>&1; tail -4 gpurun_out/time_cfg3.txt
