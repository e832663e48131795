#!/usr/bin/env bash
# the A/B switches of this round's CG / PDL / ordering changes through the kernel and solver parity tests
set -u
mkdir -p gpurun_out
T="tests/test_gpu_kernels.py tests/test_gpu_solver.py tests/test_gpu_orth.py tests/test_gpu_parity.py"
run() { echo "== $*"; env "$@" timeout 900 python -m pytest $T -q -x --timeout 300 -k "not cfg3 and not cfg4" 2>&1 | tail -2; }
run GCG_PDL=0
run GCG_CG_STAGES=2 GCG_CG_UPD_ORDER=0
run GCG_CG_STAGES=4 GCG_CG_UPD_BULK=0
run GCG_CG_STAGES=0 GCG_PDL=0 GCG_CG_UPD_BULK=0
run GCG_GRAM_INTER=1 GCG_LC_DESC=1 GCG_CG_UPD_ORDER=2
run GCG_JAC_NT=256
run GCG_JAC_NT=64
run GCG_CG_PAD=0
