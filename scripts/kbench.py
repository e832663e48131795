"""Per-kernel microbenchmarks at BASELINE shapes (development helper).

Times each device op in isolation with CUDA events (warm, back to back) and
prints achieved algorithmic GB/s / GFLOP/s vs the measured HBM peak.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_06552_b200 import device as D  # noqa: E402
from paper_2111_06552_b200 import problems as P  # noqa: E402
from paper_2111_06552_b200.operators import DeviceCsr, DeviceProblem  # noqa: E402

PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
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


def report(name, sec, nbytes, flops=0.0):
    gbs = nbytes / sec / 1e9
    print(f"{name:44s} {sec*1e6:9.1f} us  {gbs:8.1f} GB/s ({100*gbs/PEAK:5.1f}% of {PEAK:.0f})"
          + (f"  {flops/sec/1e12:6.2f} TF/s" if flops else ""), flush=True)


def main(cfgs):
    rng = np.random.default_rng(1)
    print(f"FP64 peak: DMMA {D.fp64_peak(dev, 'dmma'):.1f} TF/s, DFMA {D.fp64_peak(dev, 'dfma'):.1f} TF/s",
          flush=True)
    for cfg in cfgs:
        pr = P.baseline_problem(cfg)
        a = pr.a
        n, nnz = a.shape[0], a.nnz
        A = DeviceCsr.from_scipy(dev, a)
        bs = pr.block_size or -(-pr.num_eigen // 5)
        sx = 3 * bs if pr.moving else pr.num_eigen + 3 * bs
        m = sx + 2 * bs
        print(f"== {pr.name}: n={n} nnz={nnz} bs={bs} sx={sx} m={m}")
        V = torch.from_numpy(rng.standard_normal((n, m))).to(dev.device)
        for k in sorted({bs, sx, m}):
            X = V[:, :k]
            Y = dev.empty(n, k)
            t = timeit(lambda: D.spmm(dev, A, X, Y))
            report(f"spmm k={k} (X view ld={m})", t, 12 * nnz + 4 * (n + 1) + 16 * n * k, 2 * nnz * k)
        Xc = torch.from_numpy(rng.standard_normal((n, bs))).to(dev.device)
        Yc = dev.empty(n, bs)
        dots = dev.empty(bs)
        t = timeit(lambda: D.spmm(dev, A, Xc, Yc, gamma=-0.1, Z=Xc, dot_mode=1, W=Xc, dots=dots))
        report(f"spmm k={bs} CG form (contig, dots)", t, 12 * nnz + 4 * (n + 1) + 16 * n * bs)
        from paper_2111_06552_b200.operators import DeviceSell
        Sl = DeviceSell(A)
        t = timeit(lambda: Sl.apply(Xc, Yc, gamma=-0.1, Z=Xc, dot_mode=1, W=Xc, dots=dots))
        report(f"spmm k={bs} CG form, SELL-32-1024 ({Sl.nnz_padded / nnz:.3f}x nnz)", t,
               12 * nnz + 4 * (n + 1) + 16 * n * bs)
        for k1, k2 in [(m - bs, bs), (bs, bs), (16, 16), (m, m)]:
            G = dev.empty(k1, k2)
            Xg, Yg = V[:, :k1], V[:, m - k2:]
            t = timeit(lambda: D.gram(dev, Xg, Yg, G))
            report(f"gram {k1}x{k2}", t, 8 * n * (k1 + k2), 2 * n * k1 * k2)
        for mm, d in [(m, sx), (m, bs), (m - bs, bs), (16, 16), (m, m)]:
            Cm = torch.from_numpy(rng.standard_normal((mm, d))).to(dev.device)
            Yl = dev.empty(n, d)
            Xl = V[:, :mm]
            t = timeit(lambda: D.lincomb(dev, Xl, Cm, Yl))
            report(f"lincomb {mm}x{d}", t, 8 * n * (mm + d), 2 * n * mm * d)
        for mm in (16, 20, 40, 64, m, 2 * m):
            A0 = rng.standard_normal((mm, mm))
            Am = torch.from_numpy((A0 + A0.T) / 2).to(dev.device)
            w_ = dev.empty(mm)
            V_ = dev.empty(mm, mm)
            t = timeit(lambda: D.syev(dev, Am, w_, V_), reps=5)
            print(f"syev m={mm}: {t*1e6:9.1f} us", flush=True)
            if mm <= 64:
                q_ = dev.empty(mm, mm)
                st_ = dev.empty(4)
                t = timeit(lambda: D.svqb_prepare(dev, Am, 1e-10, q_, st_), reps=5)
                print(f"svqb_prepare m={mm}: {t*1e6:9.1f} us", flush=True)
        # block CG: one solve of 30 sweeps
        prob = DeviceProblem(dev, a)
        rhs = torch.from_numpy(rng.standard_normal((n, bs))).to(dev.device)
        from paper_2111_06552_b200.cg import block_cg

        W = V[:, sx:sx + bs]
        with D.KernelProfile(dev) as prof:
            t = timeit(lambda: block_cg(dev, prob, 0.0, rhs, W, 30, 1e-30), reps=3)
        print(f"block CG 30 sweeps k={bs}: {t*1e3:.3f} ms  ({t/30*1e6:.1f} us/sweep)")
        for kk, v in prof.result.items():
            if v["launches"]:
                print(f"   {kk:12s} {v['ms']/v['launches']*1e3:8.1f} us/launch  "
                      f"{v['bytes']/(v['ms']/1e3)/1e9:8.1f} GB/s  n={v['launches']}")
        del V


if __name__ == "__main__":
    main([int(c) for c in (sys.argv[1:] or ["2"])])
