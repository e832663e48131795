#!/usr/bin/env bash
# Round-2 evidence on one GPU (each ncu pass only after its plain command exited 0):
#  - the unmodified reference's full cfg2 solve on the host cores (background, CPU only)
#  - ncu launch list of a short bench run + --set full of the fused CG sweep SpMM
#  - FP64 tensor-pipe (DMMA) counters for the Gram / LinComb kernels
#  - compute-sanitizer racecheck / synccheck / memcheck on a small workload
set -u
mkdir -p gpurun_out
( timeout 1500 python scripts/ref_full_solve.py 2 > gpurun_out/ref_full_cfg2.json 2> gpurun_out/ref_full_cfg2.err ) &
REFPID=$!
SHORT="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$SHORT > gpurun_out/bench_short.log 2>&1 || { echo "short bench failed"; tail gpurun_out/bench_short.log; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    $SHORT > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
python scripts/launch_shares.py gpurun_out/launches_bench.csv gpurun_out/launch_shares.txt "$SHORT" | head -14
gzip -f gpurun_out/launches_bench.csv
ncu --query-metrics --chip gb100 > gpurun_out/ncu_query_metrics.txt 2>&1
grep -i -E "dmma|fp64|pipe_tensor|dfma" gpurun_out/ncu_query_metrics.txt > gpurun_out/ncu_fp64_metric_names.txt
cat gpurun_out/ncu_fp64_metric_names.txt | head -40
MET=$(grep -o -E "^(sm|smsp)__[a-z0-9_]*(dmma|fp64|tensor_op|tensor)[a-z0-9_]*" gpurun_out/ncu_query_metrics.txt | sort -u | \
      awk '{printf "%s%s.avg.pct_of_peak_sustained_active", (NR>1?",":""), $1}')
echo "metrics: $MET"
for K in gram_dmma_kernel lincomb_dmma_kernel lincomb_ts_kernel; do
  ncu --metrics gpu__time_duration.sum,$MET --clock-control none -k regex:$K -s 20 -c 3 --csv \
      $SHORT > gpurun_out/ncu_fp64_$K.csv 2> gpurun_out/ncu_fp64_$K.err
  echo "$K fp64 rc=$?"
done
ncu --set full --clock-control none --import-source on -k "regex:spmm_csr_kernel" -s 200 -c 1 \
    -o gpurun_out/full_cg_sweep $SHORT > gpurun_out/ncu_full_cg_sweep.log 2>&1
echo "cg sweep full rc=$?"
python scripts/ncu_summary.py gpurun_out/full_cg_sweep.ncu-rep > gpurun_out/ncu_sum_cg_sweep.txt 2>&1
head -40 gpurun_out/ncu_sum_cg_sweep.txt
for T in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $T --print-limit 20 python scripts/sanitize_case.py \
      > gpurun_out/sanitizer_$T.log 2>&1
  echo "sanitizer $T rc=$?"; tail -4 gpurun_out/sanitizer_$T.log
done
wait $REFPID
echo "reference full solve:"; cat gpurun_out/ref_full_cfg2.json; tail -3 gpurun_out/ref_full_cfg2.err
du -sh gpurun_out
