#!/usr/bin/env bash
# Round-end evidence on one GPU: plain bench line, then (only after it exits 0) the
# ncu launch list of a short bench run and --set full captures of the top kernels,
# summarised on the box (reports removed to stay under the gpurun copy-back limit).
set -u
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_plain.log 2>&1 || { echo "bench failed"; tail gpurun_out/bench_plain.log; exit 1; }
tail -1 gpurun_out/bench_plain.log | cut -c1-300
SHORT="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$SHORT > gpurun_out/bench_short.log 2>&1 || { echo "short bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    $SHORT > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
python scripts/launch_shares.py gpurun_out/launches_bench.csv gpurun_out/launch_shares.txt "$SHORT" > /dev/null
gzip -f gpurun_out/launches_bench.csv
for K in ${KERNELS:-spmm_csr_kernel gram_dmma_kernel lincomb_ts_kernel lincomb_dmma_kernel cg_update_kernel cg_pupdate_kernel gram_sym_kernel tridiag_kernel}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-40} -c 1 \
      -o gpurun_out/full_$K $SHORT > gpurun_out/ncu_full_$K.log 2>&1
  echo "$K rc=$?"
  python scripts/ncu_summary.py gpurun_out/full_$K.ncu-rep > gpurun_out/ncu_sum_$K.txt 2>&1
  [ "$K" = "spmm_csr_kernel" ] || rm -f gpurun_out/full_$K.ncu-rep
done
du -sh gpurun_out
