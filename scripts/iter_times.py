"""Per-iteration GPU step times of a cfg2 solve (development helper): shows which iterations /
steps get slower when the active block shrinks to odd widths."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2111_06552_b200 import SolverConfig, gcg_solve
from paper_2111_06552_b200 import problems as P, device as D
from paper_2111_06552_b200.operators import as_device_problem
pr = P.baseline_problem(2)
dev = D.default_context()
prob = as_device_problem(dev, pr.a, pr.b, validate=False)
bs = -(-pr.num_eigen // 5); sx = pr.num_eigen + 3 * bs
x0 = torch.from_numpy(np.random.Generator(np.random.PCG64(0)).standard_normal((pr.a.shape[0], sx))).to(dev.device)
cfg = SolverConfig(num_eigen=pr.num_eigen, tol=pr.tol, init="normal", residual="relative", validate=False,
                   return_device=True, collect_history=True)
gcg_solve(prob, None, cfg, x0=x0)
rep = gcg_solve(prob, None, cfg, x0=x0)
for h in rep.history:
    m = dict(h.timings) if hasattr(h, "timings") else {}
    print(h.iteration, h.num_converged, h.basis_size, h.cg_iterations,
          {k: round(1e3 * v, 3) for k, v in (m or {}).items()})
