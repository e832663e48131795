"""Timing of the dense symmetric eigensolver at the Rayleigh-Ritz orders (development
helper): full spectrum and the RR index range 1..d, eig.cu vs cuSOLVER syevd/syevdx
(run twice: default and GCG_SYEV=cusolver)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2111_06552_b200 import device as D, _lib
from paper_2111_06552_b200.dense import sym_eig_full, sym_eig_range

dev = D.default_context()
rng = np.random.default_rng(0)
tag = os.environ.get("GCG_SYEV", "eig.cu")


def timeit(f, reps=5):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for m in [int(x) for x in (sys.argv[1:] or ["200", "300", "400", "500", "700", "1000"])]:
    a = rng.standard_normal((m, m))
    a = (a + a.T) / 2
    A = torch.from_numpy(a).to(dev.device)
    t_full = timeit(lambda: sym_eig_full(dev, A))
    d = (3 * m) // 5
    t_rng = timeit(lambda: sym_eig_range(dev, A, 1, d))
    dec = sym_eig_full(dev, A)
    ww = np.linalg.eigvalsh(a)
    err = np.abs(dec.values.cpu().numpy() - ww).max() / np.abs(ww).max()
    V = dec.vectors.cpu().numpy()
    orth = np.abs(V.T @ V - np.eye(m)).max()
    print(f"{tag:9s} m={m:5d} full {t_full:8.3f} ms  range 1..{d:4d} {t_rng:8.3f} ms  "
          f"rel_err {err:.1e}  orth {orth:.1e}", flush=True)
