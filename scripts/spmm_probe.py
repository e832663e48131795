"""SpMM at the cfg2 CG shape (k = 20, contiguous X, fused shift + dots): timing / ncu target."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_06552_b200 import device as D  # noqa: E402
from paper_2111_06552_b200 import problems as P  # noqa: E402
from paper_2111_06552_b200.operators import DeviceCsr  # noqa: E402

dev = D.default_context()
a = P.laplacian_3d(int(os.environ.get("N", "64")))
n = a.shape[0]
k = int(os.environ.get("K", "20"))
A = DeviceCsr.from_scipy(dev, a)
X = torch.from_numpy(np.random.default_rng(0).standard_normal((n, k))).to(dev.device)
Y = dev.empty(n, k)
dots = dev.empty(k)
reps = int(os.environ.get("REPS", "20"))
f = lambda: D.spmm(dev, A, X, Y, gamma=-0.1, Z=X, dot_mode=1, W=X, dots=dots)
for _ in range(3):
    f()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(dev.stream)
for _ in range(reps):
    f()
e1.record(dev.stream)
torch.cuda.synchronize()
print(f"spmm CG form k={k}: {e0.elapsed_time(e1) / reps * 1e3:7.1f} us", flush=True)
