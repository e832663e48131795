set -u
mkdir -p gpurun_out
timeout 300 python scripts/eig_bench.py 200 > gpurun_out/eig_smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/eig_smoke.log | tail -5
timeout 300 python scripts/eig_bench.py 400 > gpurun_out/eig_smoke2.log 2>&1; echo "smoke400 rc=$?"; cat gpurun_out/eig_smoke2.log | tail -5
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "syev or eig or grid" > gpurun_out/eig_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/eig_tests.log
timeout 600 python scripts/eig_bench.py > gpurun_out/eig_bench.log 2>&1; echo "bench rc=$?"; cat gpurun_out/eig_bench.log
GCG_SYEV=cusolver timeout 600 python scripts/eig_bench.py > gpurun_out/eig_bench_cusolver.log 2>&1; echo "cus rc=$?"; cat gpurun_out/eig_bench_cusolver.log
timeout 600 python -m pytest tests/test_gpu_solver.py -q -x -k "cfg3" > gpurun_out/cfg3.log 2>&1; echo "cfg3 rc=$?"; tail -3 gpurun_out/cfg3.log
