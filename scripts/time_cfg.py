"""Quick timing of one BASELINE config solve on the GPU (development helper)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2111_06552_b200 import SolverConfig, gcg_solve, _lib
from paper_2111_06552_b200 import problems as P
from paper_2111_06552_b200 import device as D
from paper_2111_06552_b200.operators import as_device_problem

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
pr = P.baseline_problem(cfg)
dev = D.default_context()
prob = as_device_problem(dev, pr.a, pr.b, validate=False)
for rep_i in range(2):
    torch.cuda.synchronize()
    l0 = _lib.launch_count(); t0 = time.perf_counter()
    rep = gcg_solve(prob, None, SolverConfig(num_eigen=pr.num_eigen, block_size=pr.block_size, tol=pr.tol,
                    moving=pr.moving, seed=0, init="normal", residual="relative", max_gcg_iters=maxit,
                    return_device=True))
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"cfg{cfg} run{rep_i}: {rep.status} iters={rep.iterations} time={dt:.3f}s launches={_lib.launch_count()-l0} "
          f"maxres={rep.residuals.max():.2e} lam0={rep.eigenvalues[0]:.12f}")
    st = {k: sum(h.timings[k] for h in rep.history) for k in rep.history[0].timings}
    print("  step times:", {k: round(v, 3) for k, v in st.items()}, "cg sweeps", sum(h.cg_iterations for h in rep.history))
ex = P.analytic_eigenvalues(cfg, pr.num_eigen)
if ex is not None:
    print("  max rel err vs analytic:", np.abs(rep.eigenvalues - ex).max() / ex.max())
