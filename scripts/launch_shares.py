"""Per-kernel share of an ncu launch list (gpu__time_duration.sum CSV), dev helper."""
import collections
import csv
import sys

path, out = sys.argv[1], sys.argv[2]
cmd = sys.argv[3] if len(sys.argv) > 3 else ""
rows = list(csv.DictReader(l for l in open(path) if not l.startswith("==")))
agg, cnt = collections.Counter(), collections.Counter()
for r in rows:
    n = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").strip()
    agg[n] += float(r["Metric Value"])
    cnt[n] += 1
tot = sum(agg.values())
lines = [f"# ncu launch list of `{cmd}` (cold-cache, serialised): {len(rows)} launches, "
         f"{tot / 1e6:.1f} ms kernel time", "# share  total_ms  launches  avg_us  kernel"]
for n, v in agg.most_common(40):
    lines.append(f"{100 * v / tot:6.2f}% {v / 1e6:9.2f} {cnt[n]:8d} {v / cnt[n] / 1e3:8.1f}  {n}")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:14]))
