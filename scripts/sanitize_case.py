"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck): a cfg1-shaped
solve (Jacobi + one-CTA tridiagonal RR, DMMA Gram/LinComb, block CG, orthogonalisation)
plus the multi-CTA eigensolver path (m = 300) and a few tall-skinny shapes."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_06552_b200 import SolverConfig, gcg_solve  # noqa: E402
from paper_2111_06552_b200 import device as D  # noqa: E402
from paper_2111_06552_b200 import problems as P  # noqa: E402
from paper_2111_06552_b200.dense import sym_eig_full, sym_eig_range  # noqa: E402

rep = gcg_solve(P.laplacian_2d(30), None, SolverConfig(num_eigen=20, tol=1e-8, seed=0,
                                                       max_gcg_iters=4))
print("solve", rep.status, rep.iterations)
dev = D.default_context()
rng = np.random.default_rng(0)
for m in (120, 300):
    a = rng.standard_normal((m, m))
    A = torch.from_numpy((a + a.T) / 2).to(dev.device)
    sym_eig_full(dev, A)
    sym_eig_range(dev, A, 1, m // 2)
X = torch.from_numpy(rng.standard_normal((5000, 200))).to(dev.device)
G = dev.empty(200, 40)
D.gram(dev, X, X[:, :40], G)
Y = dev.empty(5000, 40)
D.lincomb(dev, X, G, Y)
torch.cuda.synchronize()
print("sanitize-case ok")
