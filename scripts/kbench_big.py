"""Kernel throughput at the large BASELINE configs (4: var-coef 7-pt 128^3, 5: 27-pt 256^3)
with the operators assembled in HBM by the device generators (devgen.py) and N(0,1)
multivectors drawn on the device — the host generators and a host-drawn 134 GB block are
out of reach.  Same byte/flop formulas as scripts/kbench.py.

    python scripts/kbench_big.py 4 5
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2111_06552_b200 import device as D  # noqa: E402
from paper_2111_06552_b200.devgen import device_baseline_problem  # noqa: E402

dev = D.default_context()
PEAK = 6526.5


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dev.stream)
    for _ in range(reps):
        fn()
    e1.record(dev.stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def report(name, sec, nbytes, flops=0.0):
    gbs = nbytes / sec / 1e9
    tf = f"   {flops / sec / 1e12:6.2f} TF/s" if flops else ""
    print(f"{name:44s} {sec * 1e6:10.1f} us  {gbs:8.1f} GB/s ({100 * gbs / PEAK:5.1f}% of {PEAK:.0f}){tf}",
          flush=True)


def main(cfgs):
    gen = torch.Generator(device=dev.device)
    gen.manual_seed(1)
    for cfg in cfgs:
        prob, meta = device_baseline_problem(dev, cfg)
        A = prob.A
        n, nnz = A.n, A.nnz
        bs = meta.block_size or -(-meta.num_eigen // 5)
        sx = 3 * bs if meta.moving else meta.num_eigen + 3 * bs
        print(f"== {meta.name}: n={n} nnz={nnz} bs={bs} sx={sx} (device-assembled)", flush=True)
        # V holds [X (sx) | W (bs)]: the STEP2 Gram / LinComb shapes and the CG block
        V = torch.empty(n, sx + bs, dtype=torch.float64, device=dev.device)
        V.normal_(generator=gen)
        Y = dev.empty(n, bs)
        mat = 12 * nnz + 4 * (n + 1)
        for k in (bs,):
            X = V[:, sx:sx + k]
            t = timeit(lambda: D.spmm(dev, A, X, Y))
            report(f"spmm k={k} (X view ld={sx + bs})", t, mat + 16 * n * k, 2 * nnz * k)
        Xc = V[:, sx:sx + bs].contiguous()
        dots = dev.empty(bs)
        t = timeit(lambda: D.spmm(dev, A, Xc, Y, gamma=-0.1, Z=Xc, dot_mode=1, W=Xc, dots=dots))
        report(f"spmm k={bs} CG form (contig, dots)", t, mat + 16 * n * bs)
        del Xc
        G = dev.empty(sx, bs)
        t = timeit(lambda: D.gram(dev, V[:, :sx], V[:, sx:], G), reps=5)
        report(f"gram {sx}x{bs}", t, 8 * n * (sx + bs), 2 * n * sx * bs)
        Gs = dev.empty(bs, bs)
        t = timeit(lambda: D.gram(dev, V[:, sx:], V[:, sx:], Gs), reps=5)
        report(f"gram {bs}x{bs} (X'X)", t, 8 * n * bs, 2 * n * bs * bs)
        Cm = torch.randn(sx, bs, dtype=torch.float64, device=dev.device, generator=gen)
        t = timeit(lambda: D.lincomb(dev, V[:, :sx], Cm, Y), reps=5)
        report(f"lincomb {sx}x{bs}", t, 8 * n * (sx + bs), 2 * n * sx * bs)
        del V, Y, G, Gs, prob, A
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main([int(c) for c in (sys.argv[1:] or ["4", "5"])])
