"""cProfile of the bench's end-to-end call (pinned host CSR + x0 in, host eigenvectors
out, validate=True) at cfg2: where the e2e - device-time gap goes (development helper)."""
import cProfile
import pstats
import sys
import time

import numpy as np
import scipy.sparse
import torch

sys.path.insert(0, ".")
from paper_2111_06552_b200 import SolverConfig, gcg_solve  # noqa: E402
from paper_2111_06552_b200 import problems as P  # noqa: E402

pr = P.baseline_problem(2)


def pinned(arr):
    t = torch.empty(arr.shape, dtype=torch.from_numpy(arr[:0]).dtype, pin_memory=True)
    out = t.numpy()
    out[...] = arr
    return out


src = scipy.sparse.csr_matrix(pr.a)
a = scipy.sparse.csr_matrix((pinned(src.data.astype(np.float64)), pinned(src.indices.astype(np.int32)),
                             pinned(src.indptr.astype(np.int32))), shape=src.shape)
x0 = torch.from_numpy(np.random.Generator(np.random.PCG64(0)).standard_normal((pr.a.shape[0], 160))).pin_memory()
cfg = SolverConfig(num_eigen=100, tol=1e-8, seed=0, init="normal", residual="relative", validate=True)
for _ in range(2):
    gcg_solve(a, None, cfg, x0=x0)
torch.cuda.synchronize()
t0 = time.perf_counter()
prof = cProfile.Profile()
prof.enable()
gcg_solve(a, None, cfg, x0=x0)
torch.cuda.synchronize()
prof.disable()
print(f"e2e call {1e3 * (time.perf_counter() - t0):.1f} ms")
st = pstats.Stats(prof)
st.sort_stats("cumtime").print_stats(30)
