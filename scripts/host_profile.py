"""Host-side profile of one cfg2 solve (development helper): cProfile over the solve
with the GPU running, plus the time the host spends blocked in device syncs."""
import cProfile
import pstats
import sys
import time

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
for _ in range(2):
    gcg_solve(prob, None, cfg, x0=x0)
torch.cuda.synchronize()
t0 = time.perf_counter()
gcg_solve(prob, None, cfg, x0=x0)
torch.cuda.synchronize()
print(f"plain solve wall {1e3 * (time.perf_counter() - t0):.1f} ms")
pr_ = cProfile.Profile()
pr_.enable()
gcg_solve(prob, None, cfg, x0=x0)
torch.cuda.synchronize()
pr_.disable()
st = pstats.Stats(pr_)
st.sort_stats("tottime").print_stats(45)
st.sort_stats("cumulative").print_stats(60)
