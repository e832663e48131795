"""Small symmetric Gram timing (k <= 32, X'X), dev helper."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_06552_b200 import device as D  # noqa: E402
dev = D.default_context()
def timeit(fn, reps=30):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dev.stream); [fn() for _ in range(reps)]; e1.record(dev.stream); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3
rng = np.random.default_rng(0)
n = 262144
V = torch.from_numpy(rng.standard_normal((n, 200))).to(dev.device)
out = []
for k in (8, 10, 16, 20, 32):
    X = V[:, 180 - k:180]
    G = dev.empty(k, k)
    t = timeit(lambda: D.gram(dev, X, X, G))
    out.append(f"k={k}:{t*1e6:.1f}us({8*n*k/t/1e9:.0f}GB/s)")
print(f"GCG_GRAM_SYM={os.environ.get('GCG_GRAM_SYM','1')}: " + "  ".join(out), flush=True)
