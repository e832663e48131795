"""torch.profiler (CUPTI) view of one cfg2 solve: GPU busy time by kernel vs wall (dev helper)."""
import collections
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_06552_b200 import SolverConfig, gcg_solve  # noqa: E402
from paper_2111_06552_b200 import problems as P, device as D  # noqa: E402
from paper_2111_06552_b200.operators import as_device_problem  # noqa: E402

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pr = P.baseline_problem(cfgn)
dev = D.default_context()
prob = as_device_problem(dev, pr.a, pr.b, validate=False)
bs = pr.block_size or -(-pr.num_eigen // 5)
sx = 3 * bs if pr.moving else pr.num_eigen + 3 * bs
x0 = torch.from_numpy(np.random.Generator(np.random.PCG64(0)).standard_normal((pr.a.shape[0], sx))).to(dev.device)
cfg = SolverConfig(num_eigen=pr.num_eigen, tol=pr.tol, block_size=pr.block_size, moving=pr.moving,
                   init="normal", residual="relative", validate=False, return_device=True)
gcg_solve(prob, None, cfg, x0=x0)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
t = time.perf_counter()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    rep = gcg_solve(prob, None, cfg, x0=x0)
    torch.cuda.synchronize()
wall = time.perf_counter() - t
ev = [e for e in p.events() if e.device_type == torch.autograd.DeviceType.CUDA]
agg = collections.Counter()
cnt = collections.Counter()
iv = []
for e in ev:
    name = e.name.split("(")[0].split("<")[0][:48]
    agg[name] += e.device_time
    cnt[name] += 1
    iv.append((e.time_range.start, e.time_range.end))
iv.sort()
busy, cur_s, cur_e = 0.0, None, None
for s, e_ in iv:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e_
    else:
        cur_e = max(cur_e, e_)
if cur_e is not None:
    busy += cur_e - cur_s
span = (iv[-1][1] - iv[0][0]) if iv else 0
print(f"iters {rep.iterations}  wall {wall*1e3:.1f} ms  gpu span {span/1e3:.1f} ms  busy {busy/1e3:.1f} ms  "
      f"launches {len(ev)}")
for n, v in agg.most_common(30):
    print(f"{v/1e3:9.2f} ms {cnt[n]:6d}  {v/cnt[n]:8.1f} us  {n}")

# GPU idle gaps: which kernel precedes / follows each gap (host-bound stretches)
evs = sorted(((e.time_range.start, e.time_range.end, e.name.split("(")[0].split("<")[0][-40:])
              for e in ev), key=lambda t: t[0])
gaps = collections.Counter()
gap_n = collections.Counter()
last_end, last_name = None, None
for s, e_, nm in evs:
    if last_end is not None and s - last_end > 5.0:
        key = f"{last_name} -> {nm}"
        gaps[key] += s - last_end
        gap_n[key] += 1
    if last_end is None or e_ > last_end:
        last_end, last_name = e_, nm
print("---- idle gaps > 5 us (total ms, count): preceding -> following kernel")
for k, v in gaps.most_common(25):
    print(f"{v/1e3:8.2f} ms {gap_n[k]:5d}  {k}")
