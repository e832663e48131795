"""Multivector operations of one solve: single-GPU pass-through or row-partitioned.

The solver, the B-orthogonalisation and block CG call these instead of the raw
C-ABI wrappers, so the same control flow runs on one GPU or on a row-partitioned
multi-GPU problem:

* SpMM inputs are local row blocks whose storage continues with `nghost` ghost
  rows; `spmm` first refreshes the ghost rows from the neighbours (halo
  exchange), then runs the local CSR (ghost columns index rows >= nloc);
* Gram blocks and column dots are local partial sums followed by an ordered
  all-gather sum (bit-identical on every rank, deterministic run to run — the
  paper's MPI_Allreduce of SUBMAT);
* the small dense algebra (RR, SVQB, momentum) is replicated; the RR
  eigenvectors are broadcast from rank 0 so every replica takes the same
  decisions;
* block CG runs its sweeps in the library and calls back for the halo and the
  two column-sum reductions per sweep (gcg_block_cg_dist).
"""

from __future__ import annotations

import numpy as np
import torch

from . import device as D
from .cg import CgReport

__all__ = ["LocalOps", "device_to_host_f"]

_STAGE_BYTES = 32 << 20
_stage = []  # two reusable pinned staging buffers


class PrefaultedHost:
    """The F-order host array the eigenvectors are returned in, prepared by a background
    thread while the solve runs: page-locked memory from torch's caching host allocator
    (so the final device->host copy is one DMA at full link speed, and repeated solves
    reuse the pinned blocks), else — if pinning fails — a pageable array whose pages the
    thread touches (libc memset through ctypes, which releases the GIL) so the copy does
    not pay ~50 k first-touch page faults on the critical path."""

    def __init__(self, n, k):
        import threading

        self.shape = (n, k)
        self.arr = None
        self.pinned = False
        self._thread = None
        if n * k * 8 >= (1 << 24):
            self._thread = threading.Thread(target=self._prepare, daemon=True)
            self._thread.start()
        else:
            self.arr = np.empty((n, k), order="F")

    def _prepare(self):
        n, k = self.shape
        try:
            t = torch.empty(n * k, dtype=torch.float64, pin_memory=True)
            self.arr = t.numpy().reshape((k, n)).T  # F-order view of the pinned block
            self.pinned = True
        except Exception:
            import ctypes

            self.arr = np.empty((n, k), order="F")
            libc = ctypes.CDLL(None)
            libc.memset(ctypes.c_void_p(self.arr.ctypes.data), 0, ctypes.c_size_t(self.arr.nbytes))

    def take(self, shape):
        if self._thread is not None:
            self._thread.join()
        return self.arr if self.arr is not None and self.arr.shape == tuple(shape) else None


def device_to_host_f(dev, X, out=None):
    """Device block (row-major view) -> new F-order host array, through two reused pinned
    staging buffers: the DMA of chunk i+1 overlaps the (multi-threaded) host copy of
    chunk i, and no per-call page-locking of the result is needed.  A plain .cpu() of
    the 210 MB cfg2 eigenvector block runs at ~2 GB/s (pageable staging + first-touch
    page faults); this path is bounded by the host copy."""
    n, k = X.shape
    if out is None or out.shape != (n, k) or not out.flags.f_contiguous:
        out = np.empty((n, k), order="F")
    if out.size == 0:
        return out
    torch.cuda.current_stream(X.device).wait_stream(dev.stream)
    T = X.t().contiguous()  # k x n row-major == the F-order n x k layout
    src = T.view(-1)
    dst = torch.from_numpy(out.reshape(-1, order="F"))
    total = src.numel()
    if dst.is_pinned():  # page-locked result (PrefaultedHost): one DMA, no staging
        dst.copy_(src, non_blocking=True)
        torch.cuda.current_stream(X.device).synchronize()
        return out
    chunk = _STAGE_BYTES // 8
    if total <= chunk:
        dst.copy_(src.cpu())
        return out
    if not _stage:
        _stage.extend(torch.empty(chunk, dtype=torch.float64, pin_memory=True) for _ in range(2))
    side = torch.cuda.Stream(device=X.device)
    side.wait_stream(dev.stream)
    evs = []
    with torch.cuda.stream(side):
        starts = list(range(0, total, chunk))
        for i, s in enumerate(starts[:2]):
            e = min(s + chunk, total)
            _stage[i][: e - s].copy_(src[s:e], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
            evs.append(ev)
        for i, s in enumerate(starts):
            e = min(s + chunk, total)
            evs[i].synchronize()
            dst[s:e].copy_(_stage[i % 2][: e - s])
            j = i + 2
            if j < len(starts):
                s2 = starts[j]
                e2 = min(s2 + chunk, total)
                _stage[j % 2][: e2 - s2].copy_(src[s2:e2], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(side)
                evs.append(ev)
    dev.stream.wait_stream(side)
    return out


class LocalOps:
    """One GPU, whole problem: thin pass-through to the C ABI."""

    distributed = False
    rank = 0
    size = 1

    def __init__(self, dev, prob):
        self.dev = dev
        self.prob = prob
        self.nloc = prob.n          # owned rows
        self.nghost = 0
        self.n_global = prob.n
        self.row0 = 0

    # -- allocation -----------------------------------------------------------
    def vec(self, k, zero=False):
        """n_local x k block whose storage has room for the ghost rows (SpMM input)."""
        buf = self.dev.zeros(self.nloc + self.nghost, k) if zero else \
            self.dev.empty(self.nloc + self.nghost, k)
        return buf[: self.nloc]

    # -- long-vector ops --------------------------------------------------------
    def spmm(self, op, X, Y, **kw):
        return D.spmm(self.dev, op, X, Y, **kw)

    def apply(self, op, X):
        out = self.dev.empty(X.shape[0], X.shape[1])
        return self.spmm(op, X, out)

    def gram(self, X, Y, G, **kw):
        return D.gram(self.dev, X, Y, G, **kw)

    def col_dots(self, X, Y, out):
        return D.col_dots(self.dev, X, Y, out)

    def residuals(self, AX, X, BX, lam, mode, out):
        return D.ritz_residuals(self.dev, AX, X, BX, lam, mode, out)

    def block_cg(self, vals, shift, rhs, x, max_iters, rel_tol, x0=None):
        """Block CG into x; the initial guess is x0 when given (else x's contents)."""
        k = rhs.shape[1]
        sweeps = self.dev.zeros(1, dtype=torch.int32)
        conv = self.dev.zeros(k, dtype=torch.int8)
        frozen = self.dev.zeros(k, dtype=torch.int8)
        relres = self.dev.zeros(k)
        if x0 is not None and self.distributed:
            D.copy(self.dev, x0, x)  # the row-partitioned CG reads its guess from x
            x0 = None
        if x0 is None:
            self._cg(vals, shift, rhs, x, max_iters, rel_tol, sweeps, conv, frozen, relres)
        else:
            self._cg(vals, shift, rhs, x, max_iters, rel_tol, sweeps, conv, frozen, relres, x0=x0)
        return CgReport(sweeps, conv, frozen, relres)

    def _cg(self, vals, shift, rhs, x, max_iters, rel_tol, sweeps, conv, frozen, relres, x0=None):
        D.block_cg(self.dev, self.prob.A, vals, shift, rhs, x, max_iters, rel_tol, sweeps, conv,
                   frozen, relres, x0=x0)

    # -- replicated small data ------------------------------------------------
    def broadcast(self, t):
        return t

    def allgather_sum_small(self, t):
        """Ordered sum over ranks of a replicated-shape small tensor (identity on one GPU)."""
        return t

    def host_rows(self, X, out=None):
        """Local rows of a device block as a host array (F-order)."""
        return device_to_host_f(self.dev, X, out)
