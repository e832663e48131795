"""cProfile of one cfg2 solve: where the host spends time (development helper)."""
import cProfile, pstats, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2111_06552_b200 import SolverConfig, gcg_solve
from paper_2111_06552_b200 import problems as P, device as D
from paper_2111_06552_b200.operators import as_device_problem
pr = P.baseline_problem(2)
dev = D.default_context()
prob = as_device_problem(dev, pr.a, None, validate=False)
x0 = torch.from_numpy(np.random.Generator(np.random.PCG64(0)).standard_normal((pr.a.shape[0], 160))).to(dev.device)
cfg = SolverConfig(num_eigen=100, tol=1e-8, init="normal", residual="relative", validate=False, return_device=True)
gcg_solve(prob, None, cfg, x0=x0); torch.cuda.synchronize()
t = time.perf_counter()
pr_ = cProfile.Profile(); pr_.enable()
rep = gcg_solve(prob, None, cfg, x0=x0); torch.cuda.synchronize()
pr_.disable()
print("wall", time.perf_counter() - t)
st = pstats.Stats(pr_); st.sort_stats("tottime").print_stats(18)
