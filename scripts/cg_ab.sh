#!/usr/bin/env bash
# A/B of the fused CG sweep variants on the cfg2 bench (device-timed solve).
for v in ${VARIANTS:-3 4}; do
  GCG_CG_MINB=$v python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_minb$v.log 2>&1
  python - "$v" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/ab_minb{sys.argv[1]}.log").read().strip().splitlines()[-1])
k = d["kernels"]
print(f"minb={sys.argv[1]} value={d['value']:.4f} iters={d['iterations']} spmm={k['spmm']['ms_per_step']:.1f}ms "
      f"({k['spmm']['launches_per_step']:.0f}, {k['spmm']['GBps']:.0f} GB/s) upd={k['cg_update']['ms_per_step']:.1f}ms "
      f"frac={d['roofline']['frac']:.3f}")
PY
done
