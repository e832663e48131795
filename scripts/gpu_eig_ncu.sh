#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
for M in 200 500 1000; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/eig_launch_$M.csv \
    python scripts/eig_bench.py $M > /dev/null 2>&1
python - $M <<'PY'
import csv, sys, collections
m = sys.argv[1]
rows = list(csv.DictReader(l for l in open(f"gpurun_out/eig_launch_{m}.csv") if not l.startswith("==")))
# last full-spectrum call: the launches of one sym_eig_full; aggregate all calls, divide by count of tridiag
agg, cnt = collections.Counter(), collections.Counter()
for r in rows:
    n = r["Kernel Name"].split("(")[0].replace("void ", "")[:60]
    agg[n] += float(r["Metric Value"]); cnt[n] += 1
calls = max(v for k, v in cnt.items() if "tridiag" in k)
print(f"m={m}: per-call average over {calls} eigensolves (ncu, serialised)")
for n, v in agg.most_common(20):
    print(f"  {v / calls / 1e3:9.1f} us  x{cnt[n] / calls:4.1f}  {n}")
PY
done
