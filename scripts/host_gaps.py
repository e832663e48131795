"""Host-side latency after the solver's blocking points (development helper): time
from each native orth_against / count_converged return to the next library launch."""
import sys
import time
import collections

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_06552_b200 import SolverConfig, gcg_solve, _lib  # noqa: E402
from paper_2111_06552_b200 import problems as P, device as D, solver as SV  # noqa: E402
from paper_2111_06552_b200.operators import as_device_problem  # noqa: E402

pr = P.baseline_problem(2)
dev = D.default_context()
prob = as_device_problem(dev, pr.a, pr.b, validate=False)
bs = -(-pr.num_eigen // 5)
sx = pr.num_eigen + 3 * bs
x0 = torch.from_numpy(np.random.Generator(np.random.PCG64(0)).standard_normal((pr.a.shape[0], sx))).to(dev.device)
cfg = SolverConfig(num_eigen=pr.num_eigen, tol=pr.tol, init="normal", residual="relative", validate=False,
                   return_device=True)
log = []
orig_call = _lib.call


def call(name, *a):
    t0 = time.perf_counter()
    r = orig_call(name, *a)
    log.append((name, t0, time.perf_counter()))
    return r


_lib.call = call
orig_cpu = torch.Tensor.cpu


def cpu(self, *a, **k):
    t0 = time.perf_counter()
    r = orig_cpu(self, *a, **k)
    log.append(("<tensor.cpu>", t0, time.perf_counter()))
    return r


torch.Tensor.cpu = cpu
for _ in range(2):
    gcg_solve(prob, None, cfg, x0=x0)
torch.cuda.synchronize()
log.clear()
t0 = time.perf_counter()
gcg_solve(prob, None, cfg, x0=x0)
torch.cuda.synchronize()
print(f"solve wall {1e3 * (time.perf_counter() - t0):.1f} ms, {len(log)} native calls")
gap = collections.defaultdict(list)
for (n0, s0, e0), (n1, s1, e1) in zip(log, log[1:]):
    gap[f"{n0:28s} -> {n1}"].append(s1 - e0)
tot = sum(sum(v) for v in gap.values())
print(f"host time between calls {1e3 * tot:.1f} ms")
for k, v in sorted(gap.items(), key=lambda kv: -sum(kv[1]))[:30]:
    print(f"{1e3 * sum(v):7.2f} ms {len(v):5d}x {1e6 * np.mean(v):7.1f} us  {k}")
dur = collections.defaultdict(list)
for n, s, e in log:
    dur[n].append(e - s)
print("-- time inside calls")
for k, v in sorted(dur.items(), key=lambda kv: -sum(kv[1]))[:20]:
    print(f"{1e3 * sum(v):7.2f} ms {len(v):5d}x {1e6 * np.mean(v):7.1f} us  {k}")
