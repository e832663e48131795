"""Large Gram timing (cfg3/cfg4 deflation shapes), dev helper."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_06552_b200 import device as D  # noqa: E402
dev = D.default_context()
def timeit(fn, reps=10):
    for _ in range(2): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dev.stream); [fn() for _ in range(reps)]; e1.record(dev.stream); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3
rng = np.random.default_rng(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 524288
SHAPES = ((200, 200), (400, 40), (900, 100), (360, 40), (160, 160))
if os.environ.get("SHAPES"):
    SHAPES = [tuple(int(v) for v in s.split("x")) for s in os.environ["SHAPES"].split(",")]
for k1, k2 in SHAPES:
    X = torch.from_numpy(rng.standard_normal((n, k1))).to(dev.device)
    Y = torch.from_numpy(rng.standard_normal((n, k2))).to(dev.device)
    G = dev.empty(k1, k2)
    t = timeit(lambda: D.gram(dev, X, Y, G))
    C = torch.from_numpy(rng.standard_normal((k1, k2))).to(dev.device)
    Z = dev.empty(n, k2)
    tl = timeit(lambda: D.lincomb(dev, X, C, Z))
    print(f"n={n} {k1}x{k2}: gram {t*1e3:.3f} ms {2*n*k1*k2/t/1e12:.2f} TF/s | lincomb {tl*1e3:.3f} ms "
          f"{2*n*k1*k2/tl/1e12:.2f} TF/s", flush=True)
    del X, Y, Z
