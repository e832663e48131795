#!/usr/bin/env bash
# Round-2 evidence of the current state (each ncu pass only after its plain run exited 0):
# bench line (default args), ncu launch list of a short bench, --set full of the fused
# CG sweep SpMM and the r-update, kbench at cfg2 and the large configs.
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_default.log | cut -c1-600
SHORT="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$SHORT > gpurun_out/bench_short.log 2>&1 || { echo "short bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    $SHORT > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
python scripts/launch_shares.py gpurun_out/launches_bench.csv gpurun_out/launch_shares.txt "$SHORT" | head -16
gzip -f gpurun_out/launches_bench.csv
SKIP=200 bash scripts/ncu_cg.sh
head -24 gpurun_out/ncu_sum_cg_sweep.txt; head -24 gpurun_out/ncu_sum_cg_update.txt
rm -f gpurun_out/full_cg_sweep.ncu-rep
timeout 600 python scripts/kbench.py 2 > gpurun_out/kbench2.log 2>&1; echo "kbench rc=$?"; cat gpurun_out/kbench2.log | head -40
timeout 900 python scripts/kbench_big.py 4 5 > gpurun_out/kbench_big.log 2>&1; echo "kbench_big rc=$?"; cat gpurun_out/kbench_big.log
du -sh gpurun_out
