"""Where the end-to-end (host buffers) time goes beyond the device solve (dev helper)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2111_06552_b200 import SolverConfig, gcg_solve
from paper_2111_06552_b200 import problems as P, device as D
from paper_2111_06552_b200.operators import as_device_problem

pr = P.baseline_problem(2)
dev = D.default_context()
x0 = np.random.Generator(np.random.PCG64(0)).standard_normal((pr.a.shape[0], 160))
x0_pin = torch.from_numpy(x0).pin_memory()
cfg = SolverConfig(num_eigen=100, tol=1e-8, seed=0, init="normal", residual="relative", validate=False)
for rep_i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    prob = as_device_problem(dev, pr.a, None, validate=False)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    xd = x0_pin.to(dev.device, non_blocking=True)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    cfg.return_device = True
    rep = gcg_solve(prob, None, cfg, x0=xd)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    from paper_2111_06552_b200.mvops import LocalOps
    h = LocalOps(dev, prob).host_rows(rep.eigenvectors)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    cfg.return_device = False
    rep2 = gcg_solve(pr.a, None, cfg, x0=x0_pin)
    torch.cuda.synchronize(); t5 = time.perf_counter()
    print(f"upload A {1e3*(t1-t0):.1f} ms | x0 H2D {1e3*(t2-t1):.1f} | solve(dev) {1e3*(t3-t2):.1f} | "
          f"evec D2H {1e3*(t4-t3):.1f} | full public call {1e3*(t5-t4):.1f} ms", flush=True)
