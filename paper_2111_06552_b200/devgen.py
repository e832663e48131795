"""BASELINE operators assembled directly in HBM.

Device counterparts of problems.py: ``stencil_csr`` and the config 1/2/4/5
generators write row pointers, column indices and values with library kernels
(gcg_stencil_csr, gcg_varcoef7_weights; csrc/gen.cu) — bit-identical to the host
generators, without the host temporaries (config 5: 450 M nonzeros) or the H2D
copy.  The variable-coefficient field of config 4 is drawn on the host with the
same seeded PCG64 stream as problems.varcoef_diffusion_3d (n doubles uploaded),
the faces and the diagonal are computed on the device.  Config 3 (P1 FEM) is
assembled on the host (problems.fem_p1_cube) and uploaded.
"""

from __future__ import annotations

import ctypes as C
import itertools

import numpy as np
import torch

from . import _lib
from . import device as D
from . import problems as P
from .errors import InvalidShape
from .operators import DeviceCsr, DeviceProblem

__all__ = ["stencil_device", "stencil_slab_device", "baseline_stencil_spec", "laplacian_2d_device",
           "laplacian_3d_device", "stencil27_device", "varcoef_diffusion_3d_device",
           "device_baseline_problem"]


def _grid3(shape, offsets):
    shape = tuple(int(s) for s in shape)
    if len(shape) == 2:
        return (1,) + shape, [(0,) + tuple(o) for o in offsets]
    if len(shape) == 3:
        return shape, [tuple(o) for o in offsets]
    raise InvalidShape(f"stencil grids are 2-D or 3-D, got {shape}")


def stencil_device(ctx, shape, offsets, weights):
    """DeviceCsr of a constant- or per-row-coefficient stencil (problems.stencil_csr)."""
    (n0, n1, n2), offs = _grid3(shape, offsets)
    noff = len(offs)
    n = n0 * n1 * n2
    flat = (C.c_int32 * (3 * noff))(*[v for o in offs for v in o])
    nnz = C.c_int64()
    _lib.check(_lib.load().gcg_stencil_nnz(n0, n1, n2, noff, flat, C.byref(nnz)), "gcg_stencil_nnz")
    keep = []  # temporaries that must outlive the launch
    wc, wr = _weight_args(ctx, weights, n, keep)
    rowptr = ctx.empty(n + 1, dtype=torch.int32)
    colidx = ctx.empty(int(nnz.value), dtype=torch.int32)
    val = ctx.empty(int(nnz.value))
    _lib.call("gcg_stencil_csr", ctx.h, n0, n1, n2, noff, flat, wc, wr, D._p(rowptr),
              D._p(colidx), D._p(val))
    return DeviceCsr(ctx, rowptr, colidx, val, n)


def _weight_args(ctx, weights, n, keep):
    """(constant weights, per-row pointer array or None) for the stencil generators."""
    noff = len(weights)
    per_row = any(isinstance(w, torch.Tensor) for w in weights)
    wc = (C.c_double * noff)(*[0.0 if isinstance(w, torch.Tensor) else float(w) for w in weights])
    if not per_row:
        return wc, None
    ptrs = []
    for w in weights:
        if isinstance(w, torch.Tensor):
            if w.shape != (n,) or w.dtype != torch.float64 or not w.is_cuda:
                raise InvalidShape("per-row stencil weights must be (n,) float64 device arrays")
            ptrs.append(w.data_ptr())
        else:
            t = ctx.empty(n)
            D.fill(ctx, t.view(n, 1), float(w))
            keep.append(t)
            ptrs.append(t.data_ptr())
    return wc, (C.c_void_p * noff)(*ptrs)


def stencil_slab_device(ctx, shape, offsets, weights, row0, row1):
    """This rank's z-slab [row0, row1) of the stencil in the local layout of a
    row-partitioned run (gcg_stencil_slab): a DeviceCsr with n = row1 - row0 owned rows
    whose columns index owned rows, then the ghost plane below, then the one above —
    the matrix distributed.local_part cuts from the global CSR, without ever building
    it.  Returns (csr, nprev, nnext)."""
    (n0, n1, n2), offs = _grid3(shape, offsets)
    noff = len(offs)
    n = n0 * n1 * n2
    flat = (C.c_int32 * (3 * noff))(*[v for o in offs for v in o])
    keep = []
    wc, wr = _weight_args(ctx, weights, n, keep)
    nloc = int(row1 - row0)
    rowptr = ctx.empty(nloc + 1, dtype=torch.int32)
    nnz = C.c_int64()
    _lib.call("gcg_stencil_slab", ctx.h, n0, n1, n2, noff, flat, wc, wr, int(row0), int(row1),
              D._p(rowptr), None, None, C.byref(nnz))
    colidx = ctx.empty(int(nnz.value), dtype=torch.int32)
    val = ctx.empty(int(nnz.value))
    ng = C.c_int64()
    _lib.call("gcg_stencil_slab", ctx.h, n0, n1, n2, noff, flat, wc, wr, int(row0), int(row1),
              D._p(rowptr), D._p(colidx), D._p(val), C.byref(ng))
    plane = n1 * n2 if n0 > 1 else n2
    nprev = min(plane, int(row0)) if row0 > 0 else 0
    nnext = min(plane, n - int(row1)) if row1 < n else 0
    assert nprev + nnext == int(ng.value)
    return DeviceCsr(ctx, rowptr, colidx, val, nloc), nprev, nnext


def baseline_stencil_spec(ctx, cfg, scale=None):
    """(grid shape, offsets, weights) of BASELINE config 1, 2, 4 or 5 (weights of config 4
    are per-row device arrays of the global grid)."""
    meta = P.baseline_problem(cfg, scale=scale, build=False)
    N = meta.grid[0]
    if cfg == 1:
        return (N, N), [(0, 0)] + _axis_offsets(2), [4.0] + [-1.0] * 4, meta
    if cfg == 2:
        return (N, N, N), [(0, 0, 0)] + _axis_offsets(3), [6.0] + [-1.0] * 6, meta
    if cfg == 4:
        rng = np.random.default_rng(0)
        kc = torch.from_numpy(np.exp(rng.standard_normal((N, N, N))).reshape(-1)).to(ctx.device)
        w = ctx.empty(7, N ** 3)
        _lib.call("gcg_varcoef7_weights", ctx.h, N, D._p(kc), D._p(w))
        return (N, N, N), [(0, 0, 0)] + _axis_offsets(3), [w[t] for t in range(7)], meta
    if cfg == 5:
        offs = list(itertools.product((-1, 0, 1), repeat=3))
        return (N, N, N), offs, [26.0 if o == (0, 0, 0) else -1.0 for o in offs], meta
    raise InvalidShape(f"config {cfg} is not a structured-grid stencil")


def _axis_offsets(nd):
    offs = []
    for ax in range(nd):
        for s in (-1, 1):
            o = [0] * nd
            o[ax] = s
            offs.append(tuple(o))
    return offs


def laplacian_2d_device(ctx, N):
    return stencil_device(ctx, (N, N), [(0, 0)] + _axis_offsets(2), [4.0] + [-1.0] * 4)


def laplacian_3d_device(ctx, N):
    return stencil_device(ctx, (N, N, N), [(0, 0, 0)] + _axis_offsets(3), [6.0] + [-1.0] * 6)


def stencil27_device(ctx, N):
    offs = list(itertools.product((-1, 0, 1), repeat=3))
    return stencil_device(ctx, (N, N, N), offs, [26.0 if o == (0, 0, 0) else -1.0 for o in offs])


def varcoef_diffusion_3d_device(ctx, N, seed=0):
    """problems.varcoef_diffusion_3d with the faces/diagonal computed on the device."""
    rng = np.random.default_rng(seed)
    kc = torch.from_numpy(np.exp(rng.standard_normal((N, N, N))).reshape(-1)).to(ctx.device)
    n = N ** 3
    w = ctx.empty(7, n)
    _lib.call("gcg_varcoef7_weights", ctx.h, N, D._p(kc), D._p(w))
    offs = [(0, 0, 0)] + _axis_offsets(3)
    return stencil_device(ctx, (N, N, N), offs, [w[t] for t in range(7)])


def device_baseline_problem(ctx, cfg, scale=None):
    """(DeviceProblem, Problem metadata without host matrices) of BASELINE config `cfg`."""
    meta = P.baseline_problem(cfg, scale=scale, build=False)
    N = meta.grid[0]
    if cfg == 1:
        A = laplacian_2d_device(ctx, N)
    elif cfg == 2:
        A = laplacian_3d_device(ctx, N)
    elif cfg == 4:
        A = varcoef_diffusion_3d_device(ctx, N)
    elif cfg == 5:
        A = stencil27_device(ctx, N)
    else:
        full = P.baseline_problem(cfg, scale=scale)
        return DeviceProblem(ctx, full.a, full.b), full
    return DeviceProblem.from_device(ctx, A), meta

