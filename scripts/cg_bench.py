"""Block-CG sweep timing at a BASELINE shape (development helper): 30 sweeps of
gcg_block_cg on the device-assembled operator with k = bs random right-hand sides.
    python scripts/cg_bench.py 4"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2111_06552_b200 import device as D  # noqa: E402
from paper_2111_06552_b200.devgen import device_baseline_problem  # noqa: E402

dev = D.default_context()
for cfg in [int(c) for c in (sys.argv[1:] or ["2", "4"])]:
    prob, meta = device_baseline_problem(dev, cfg)
    n = prob.A.n
    k = meta.block_size or -(-meta.num_eigen // 5)
    k = int(os.environ.get("CG_BENCH_K", k))
    g = torch.Generator(device=dev.device)
    g.manual_seed(0)
    rhs = torch.randn(n, k, dtype=torch.float64, device=dev.device, generator=g)
    x = torch.zeros(n, k, dtype=torch.float64, device=dev.device)
    sw = dev.zeros(1, dtype=torch.int32)
    cv = dev.zeros(k, dtype=torch.int8)
    fr = dev.zeros(k, dtype=torch.int8)
    rr = dev.zeros(k)
    run = lambda: D.block_cg(dev, prob.A, prob.A.val, -1e-3, rhs, x, 30, 1e-300, sw, cv, fr, rr)
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dev.stream)
    for _ in range(3):
        run()
    e1.record(dev.stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"cfg{cfg} n={n} k={k}: 30 sweeps {ms:.3f} ms = {ms / 30 * 1e3:.1f} us/sweep (sweeps={int(sw.item())}) "
          f"x-sha1={hashlib.sha1(x.cpu().numpy().tobytes()).hexdigest()[:10]}",
          flush=True)
    del prob, rhs, x
    torch.cuda.empty_cache()
