"""GPU idle-gap histogram over one whole cfg2 solve (development helper): every gap
between consecutive device activities, attributed to the (previous, next) activity
names, summed over the solve."""
import collections
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_06552_b200 import SolverConfig, gcg_solve  # noqa: E402
from paper_2111_06552_b200 import problems as P, device as D  # noqa: E402
from paper_2111_06552_b200.operators import as_device_problem  # noqa: E402

pr = P.baseline_problem(2)
dev = D.default_context()
prob = as_device_problem(dev, pr.a, pr.b, validate=False)
bs = -(-pr.num_eigen // 5)
sx = pr.num_eigen + 3 * bs
x0 = torch.from_numpy(np.random.Generator(np.random.PCG64(0)).standard_normal((pr.a.shape[0], sx))).to(dev.device)
cfg = SolverConfig(num_eigen=pr.num_eigen, tol=pr.tol, init="normal", residual="relative", validate=False,
                   return_device=True)
gcg_solve(prob, None, cfg, x0=x0)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as p:
    gcg_solve(prob, None, cfg, x0=x0)
    torch.cuda.synchronize()
ev = sorted(((e.time_range.start, e.time_range.end, e.name.split("(")[0].split("<")[0].replace("void ", "")[-30:])
            for e in p.events() if e.device_type == torch.autograd.DeviceType.CUDA))
gaps = collections.Counter()
cnt = collections.Counter()
last_end, last_name = ev[0][1], ev[0][2]
tot = 0.0
for s, e, nm in ev[1:]:
    g = s - last_end
    if g > 0:
        key = f"{last_name:30s} -> {nm}"
        gaps[key] += g
        cnt[key] += 1
        tot += g
    if e >= last_end:
        last_end, last_name = e, nm
print(f"total idle {tot / 1e3:.2f} ms over {len(ev)} activities, span {(ev[-1][1] - ev[0][0]) / 1e3:.2f} ms")
for k, v in gaps.most_common(30):
    print(f"{v / 1e3:8.2f} ms  {cnt[k]:6d}x  {v / cnt[k]:7.1f} us  {k}")
