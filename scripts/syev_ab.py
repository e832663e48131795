"""A/B timing of the dense symmetric eigensolvers (development helper)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2111_06552_b200 import device as D, _lib
import ctypes as C
dev = D.default_context()
rng = np.random.default_rng(0)
for m in (16, 20, 40, 64, 100, 200, 400):
    a = rng.standard_normal((m, m)); a = (a + a.T) / 2
    A = torch.from_numpy(a).to(dev.device)
    w = dev.empty(m); V = dev.empty(m, m)
    f = lambda: _lib.call("gcg_syev", dev.h, m, D._p(A), m, D._p(w), D._p(V), m) if m <= 64 else \
        _lib.call("gcg_syev", dev.h, m, D._p(A), m, D._p(w), D._p(V), m)
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [f() for _ in range(5)]; e1.record(); torch.cuda.synchronize()
    ww = np.linalg.eigvalsh(a)
    err = np.abs(w.cpu().numpy() - ww).max()
    print(f"{os.environ.get('GCG_SYEV','default'):8s} m={m:4d} {e0.elapsed_time(e1)/5*1e3:9.1f} us  err={err:.1e}", flush=True)
# index-range solver (syevdx) for the RR shapes: 1..d of m
for m, d in ((200, 160), (400, 320), (500, 300)):
    a = rng.standard_normal((m, m)); a = (a + a.T) / 2
    A = torch.from_numpy(a).to(dev.device)
    w = dev.empty(d); V = dev.empty(m, d)
    f = lambda: D.syev_range(dev, A, 1, d, w, V)
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [f() for _ in range(5)]; e1.record(); torch.cuda.synchronize()
    print(f"syevdx   m={m:4d} 1..{d} {e0.elapsed_time(e1)/5*1e3:9.1f} us", flush=True)
