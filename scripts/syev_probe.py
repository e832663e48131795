"""One dense eigensolve of order M (default 200) for ncu launch lists (dev helper)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_06552_b200 import device as D  # noqa: E402

dev = D.default_context()
m = int(os.environ.get("M", "200"))
kind = os.environ.get("KIND", "random")
rng = np.random.default_rng(m)
if kind == "random":
    a = rng.standard_normal((m, m))
    a = (a + a.T) / 2
else:  # RR-like: sorted small Ritz values coupled to a 40-wide block
    d = m - 40
    a = np.zeros((m, m))
    a[:d, :d] = np.diag(np.sort(rng.uniform(0.006, 0.3, d)))
    b = 1e-2 * rng.standard_normal((m - d, d))
    c = rng.standard_normal((m - d, m - d))
    a[d:, :d] = b
    a[:d, d:] = b.T
    a[d:, d:] = 0.05 * (c + c.T) + 0.5 * np.eye(m - d)
A = torch.from_numpy(a).to(dev.device)
w = dev.empty(m)
v = dev.empty(m, m)
for _ in range(int(os.environ.get("REPS", "2"))):
    D.syev(dev, A, w, v)
torch.cuda.synchronize()
print("max |dlambda|", np.abs(w.cpu().numpy() - np.linalg.eigvalsh(a)).max())
