"""Tall-skinny LinComb / Gram rate vs n (L2-resident vs HBM-streamed), dev helper."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_06552_b200 import device as D  # noqa: E402

dev = D.default_context()


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dev.stream)
    for _ in range(reps):
        fn()
    e1.record(dev.stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


rng = np.random.default_rng(0)
for n in (16384, 65536, 262144, 1048576):
    for m, d in ((200, 20), (180, 20), (40, 20), (200, 160)):
        X = torch.from_numpy(rng.standard_normal((n, m))).to(dev.device)
        Cm = torch.from_numpy(rng.standard_normal((m, d))).to(dev.device)
        Y = dev.empty(n, d)
        t = timeit(lambda: D.lincomb(dev, X, Cm, Y))
        G = dev.empty(m, d)
        Yg = torch.from_numpy(rng.standard_normal((n, d))).to(dev.device)
        tg = timeit(lambda: D.gram(dev, X, Yg, G))
        print(f"n={n:8d} m={m:3d} d={d:3d}  lincomb {t*1e6:8.1f} us {2*n*m*d/t/1e12:6.2f} TF/s "
              f"{8*n*(m+d)/t/1e9:7.0f} GB/s | gram {tg*1e6:8.1f} us {2*n*m*d/tg/1e12:6.2f} TF/s "
              f"{8*n*(m+d)/tg/1e9:7.0f} GB/s", flush=True)
        del X, Y, Yg
