"""Ordered GPU event trace (kernel, start gap, duration) of GCG iterations it0..it1 of one
cfg2 solve — where the idle gaps sit (development helper)."""
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
with profile(activities=[ProfilerActivity.CUDA]) as p:
    gcg_solve(prob, None, cfg, x0=x0)
    torch.cuda.synchronize()
ev = sorted(((e.time_range.start, e.time_range.end, e.name.split("(")[0].split("<")[0][-34:])
            for e in p.events() if e.device_type == torch.autograd.DeviceType.CUDA))
# iteration boundaries: the tridiag kernel marks each RR
marks = [i for i, e in enumerate(ev) if "tridiag" in e[2]]
it0, it1 = int(sys.argv[1]) if len(sys.argv) > 1 else 20, int(sys.argv[2]) if len(sys.argv) > 2 else 21
lo, hi = marks[it0], marks[it1]
last = ev[lo - 1][1]
tot_gap = 0.0
for s, e, nm in ev[lo:hi]:
    gap = s - last
    tot_gap += max(gap, 0)
    if gap > 3 or e - s > 30 or len(sys.argv) > 3:
        print(f"gap {gap:7.1f} us  dur {e - s:7.1f} us  {nm}")
    last = max(last, e)
print(f"iteration span {ev[hi][0] - ev[lo][0]:.1f} us, idle {tot_gap:.1f} us, events {hi - lo}")
# whole-solve summary: span, busy (union of kernel intervals), idle
busy, cur_s, cur_e = 0.0, None, None
for s, e, nm in ev:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
span = ev[-1][1] - ev[0][0]
print(f"solve: span {span / 1e3:.2f} ms  busy {busy / 1e3:.2f} ms  idle {(span - busy) / 1e3:.2f} ms  "
      f"kernels {len(ev)}  iteration-{it0} gaps {tot_gap:.1f} us")
