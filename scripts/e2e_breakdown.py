"""Where the end-to-end (host buffers in, host eigenvectors out) time goes at cfg2 (dev helper)."""
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
sx = 160
x0 = torch.from_numpy(np.random.Generator(np.random.PCG64(0)).standard_normal((pr.a.shape[0], sx))).pin_memory()
cfg = SolverConfig(num_eigen=100, tol=1e-8, init="normal", residual="relative", validate=False)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prob = as_device_problem(dev, pr.a, None, validate=False)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = gcg_solve(prob, None, cfg, x0=x0)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    r2 = gcg_solve(prob, None, SolverConfig(num_eigen=100, tol=1e-8, init="normal", residual="relative",
                                            validate=False, return_device=True), x0=x0)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"problem upload {1e3*(t1-t0):.1f} ms | solve host-out {1e3*(t2-t1):.1f} ms | "
          f"solve device-out {1e3*(t3-t2):.1f} ms", flush=True)
