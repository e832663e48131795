"""SpMM A/B microbench at the BASELINE shapes (env knobs GCG_SPMM_VEC / GCG_SPMM_ORDER)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_06552_b200 import device as D  # noqa: E402
from paper_2111_06552_b200 import problems as P  # noqa: E402
from paper_2111_06552_b200.operators import DeviceCsr  # noqa: E402

dev = D.default_context()


def timeit(fn, reps=30):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dev.stream)
    for _ in range(reps):
        fn()
    e1.record(dev.stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


tag = f"vec={os.environ.get('GCG_SPMM_VEC', '4')} order={os.environ.get('GCG_SPMM_ORDER', '1')}"
rng = np.random.default_rng(0)
for cfg in [int(c) for c in (sys.argv[1:] or ["2", "3"])]:
    pr = P.baseline_problem(cfg)
    a = pr.a
    n = a.shape[0]
    A = DeviceCsr.from_scipy(dev, a)
    bs = pr.block_size or -(-pr.num_eigen // 5)
    m = (3 * bs if pr.moving else pr.num_eigen + 3 * bs) + 2 * bs
    V = torch.from_numpy(rng.standard_normal((n, m))).to(dev.device)
    Xc = V[:, :bs].contiguous()
    Y = dev.empty(n, m)
    dots = dev.empty(bs)
    res = []
    res.append(("cg", timeit(lambda: D.spmm(dev, A, Xc, Y[:, :bs].view(n, bs) if False else Y[:, :bs],
                                            gamma=-0.1, Z=Xc, dot_mode=1, W=Xc, dots=dots))))
    Yc = dev.empty(n, bs)
    res.append(("cgc", timeit(lambda: D.spmm(dev, A, Xc, Yc, gamma=-0.1, Z=Xc, dot_mode=1, W=Xc,
                                             dots=dots))))
    res.append((f"view{bs}", timeit(lambda: D.spmm(dev, A, V[:, m - bs:], Yc))))
    res.append((f"view{m}", timeit(lambda: D.spmm(dev, A, V, Y))))
    print(f"{pr.name:18s} {tag}: " + "  ".join(f"{k}={v:7.1f}us" for k, v in res), flush=True)
    del V, Y
