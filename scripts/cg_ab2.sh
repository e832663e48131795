#!/usr/bin/env bash
# A/B of environment switches on the cfg2 bench: each argument is "NAME=VALUE ..." (quoted)
for cfg in "$@"; do
  env $cfg python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.log 2>&1
  python - "$cfg" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.log").read().strip().splitlines()[-1])
k = d["kernels"]
sp = k["spmm"]
print(f"[{sys.argv[1]}] value={d['value']:.4f} iters={d['iterations']} spmm={sp['ms_per_step']:.1f}ms "
      f"/{sp['launches_per_step']:.0f} = {1e3*sp['ms_per_step']/sp['launches_per_step']:.1f}us ({sp['GBps']:.0f} GB/s) "
      f"upd={k['cg_update']['ms_per_step']:.1f}ms frac={d['roofline']['frac']:.3f}", flush=True)
PY
done
