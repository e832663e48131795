"""cProfile of one BASELINE solve: where the host spends time (development helper)."""
import cProfile, pstats, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2111_06552_b200 import SolverConfig, gcg_solve
from paper_2111_06552_b200 import problems as P, device as D
from paper_2111_06552_b200.operators import as_device_problem
cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pr = P.baseline_problem(cfgn)
dev = D.default_context()
prob = as_device_problem(dev, pr.a, pr.b, validate=False)
bs = pr.block_size or -(-pr.num_eigen // 5)
sx = 3 * bs if pr.moving else pr.num_eigen + 3 * bs
x0 = torch.from_numpy(np.random.Generator(np.random.PCG64(0)).standard_normal((pr.a.shape[0], sx))).to(dev.device)
cfg = SolverConfig(num_eigen=pr.num_eigen, tol=pr.tol, block_size=pr.block_size, moving=pr.moving,
                   init="normal", residual="relative", validate=False, return_device=True)
gcg_solve(prob, None, cfg, x0=x0); torch.cuda.synchronize()
t = time.perf_counter()
pr_ = cProfile.Profile(); pr_.enable()
rep = gcg_solve(prob, None, cfg, x0=x0); torch.cuda.synchronize()
pr_.disable()
print("wall", time.perf_counter() - t)
st = pstats.Stats(pr_); st.sort_stats("tottime").print_stats(14)
st.sort_stats("cumtime").print_stats(22)
