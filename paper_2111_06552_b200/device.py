"""Device context and thin typed wrappers over the C ABI.

PyTorch is used only for device memory and the stream; every arithmetic
operation on a multivector goes through libgcgb200.so.  Multivectors are 2-D
row-major float64 tensors (or column-range views of one, stride (ld, 1)), so
a column range is a pointer offset with the parent's leading dimension.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import torch

from . import _lib
from .errors import InvalidShape

_tls = threading.local()


def _require_cuda():
    if not torch.cuda.is_available():
        raise _lib.DeviceError(
            "no CUDA device: the B200 path has no CPU fallback (run on a GPU box)"
        )


class Context:
    """One gcg context bound to a torch CUDA stream on one device."""

    def __init__(self, device=None, stream=None):
        _require_cuda()
        lib = _lib.load()
        self.device = torch.device("cuda") if device is None else torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        with torch.cuda.device(self.device):
            self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
            h = C.c_void_p()
            _lib.check(lib.gcg_ctx_create(C.byref(h), C.c_void_p(self.stream.cuda_stream)),
                       "gcg_ctx_create")
        self.h = h
        self.lib = lib

    def close(self):
        if self.h:
            self.lib.gcg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        self.stream.synchronize()

    # -- allocation helpers ------------------------------------------------
    def empty(self, *shape, dtype=torch.float64):
        return torch.empty(*shape, dtype=dtype, device=self.device)

    def zeros(self, *shape, dtype=torch.float64):
        return torch.zeros(*shape, dtype=dtype, device=self.device)

    def upload(self, arr, dtype=None):
        t = torch.from_numpy(np.ascontiguousarray(arr))
        if dtype is not None:
            t = t.to(dtype)
        return t.to(self.device, non_blocking=False)


PROF_CLASSES = ("spmm", "gram", "lincomb", "cg_update", "cg_xout", "cg_sweep")


class KernelProfile:
    """Live CUDA-event timing of the library's hot kernels on the ctx stream.

        with KernelProfile(ctx) as prof: ...      # prof.result after exit
    result[cls] = {"ms": total ms, "launches": n, "bytes": algorithmic HBM bytes}.
    """

    def __init__(self, ctx, sample=1):
        self.ctx = ctx
        self.sample = int(sample)
        self.result = None

    def __enter__(self):
        _lib.call("gcg_prof_sample", self.ctx.h, self.sample)
        _lib.call("gcg_prof_begin", self.ctx.h)
        return self

    def __exit__(self, *exc):
        out = (C.c_double * (3 * len(PROF_CLASSES)))()
        _lib.call("gcg_prof_end", self.ctx.h, out)
        _lib.call("gcg_prof_sample", self.ctx.h, 1)
        # with sampling, ms / launches / bytes cover the timed launches (every
        # `sample`-th of each class); rates (bytes / ms) are unaffected
        self.result = {
            name: {"ms": out[3 * i], "launches": int(out[3 * i + 1]), "bytes": out[3 * i + 2],
                   "sample": self.sample}
            for i, name in enumerate(PROF_CLASSES)
        }
        return False


def default_context():
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context()
        _tls.ctx = ctx
    return ctx


# ---------------------------------------------------------------------------
# typed wrappers (pointers from torch tensors; ld = stride(0) of a 2-D view)


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _ld(t):
    if t is None:
        return 0
    if t.dim() == 1:
        return 1
    if t.stride(1) != 1 and t.shape[1] > 1:
        raise InvalidShape("multivector views must be row-major (unit column stride)")
    return max(t.stride(0), t.shape[1])


def spmm(ctx, A, X, Y, alpha=1.0, gamma=0.0, Z=None, beta=0.0, Yin=None, dot_mode=0, W=None,
         dots=None, vals=None):
    """Y = alpha*(A X) + gamma*Z + beta*Yin ; optional fused column dots (gcg_spmm_csr)."""
    n, k = Y.shape
    if k == 0 or n == 0:
        return Y
    if X.shape != (A.n, k):
        raise InvalidShape(f"spmm: X {tuple(X.shape)} vs operator dim {A.n}, {k} cols")
    v = A.val if vals is None else vals
    _lib.call("gcg_spmm_csr", ctx.h, n, A.nnz, _p(A.rowptr), _p(A.colidx), _p(v), k, _p(X), _ld(X),
              float(alpha), float(gamma), _p(Z), _ld(Z), float(beta), _p(Yin), _ld(Yin), _p(Y),
              _ld(Y), int(dot_mode), _p(W), _ld(W), _p(dots))
    return Y


def gram(ctx, X, Y, G, alpha=1.0, beta=0.0, T=None, dots=None, transpose_out=False):
    """G = alpha X'Y + beta G (G row-major k1 x k2 view, or its transpose)."""
    n, k1 = X.shape
    k2 = Y.shape[1]
    if G.dim() != 2:
        raise InvalidShape("gram: G must be 2-D")
    if transpose_out:
        grs, gcs = G.stride(1), G.stride(0)
    else:
        grs, gcs = G.stride(0), G.stride(1)
    _lib.call("gcg_gram", ctx.h, n, k1, k2, _p(X), _ld(X), _p(Y), _ld(Y), float(alpha),
              float(beta), _p(G), grs, gcs, _p(T), _ld(T), _p(dots))
    return G


def lincomb(ctx, X, Cm, Y, alpha=1.0, beta=0.0):
    """Y = alpha X C + beta Y  (gcg_lincomb); Y may alias X only row-for-row
    (in place, d <= 256 — see gcgb200.h)."""
    n, m = X.shape
    d = Cm.shape[1]
    if Cm.shape[0] != m or Y.shape != (n, d):
        raise InvalidShape(f"lincomb shapes {tuple(X.shape)} {tuple(Cm.shape)} {tuple(Y.shape)}")
    _lib.call("gcg_lincomb", ctx.h, n, m, d, float(alpha), _p(X), _ld(X), _p(Cm), _ld(Cm),
              float(beta), _p(Y), _ld(Y))
    return Y


def axpby(ctx, alpha, X, beta, Y):
    n, k = Y.shape
    _lib.call("gcg_axpby", ctx.h, n, k, float(alpha), _p(X), _ld(X), float(beta), _p(Y), _ld(Y))
    return Y


def copy(ctx, X, Y):
    n, k = Y.shape
    if X.shape != Y.shape:
        raise InvalidShape(f"copy shapes {tuple(X.shape)} vs {tuple(Y.shape)}")
    _lib.call("gcg_copy", ctx.h, n, k, _p(X), _ld(X), _p(Y), _ld(Y))
    return Y


def fill(ctx, Y, value=0.0):
    n, k = Y.shape
    _lib.call("gcg_fill", ctx.h, n, k, float(value), _p(Y), _ld(Y))
    return Y


def col_scale(ctx, s, X):
    n, k = X.shape
    _lib.call("gcg_col_scale", ctx.h, n, k, _p(s), _p(X), _ld(X))
    return X


def col_dots(ctx, X, Y, out):
    n, k = X.shape
    _lib.call("gcg_col_dots", ctx.h, n, k, _p(X), _ld(X), _p(Y), _ld(Y), _p(out))
    return out


def syev(ctx, A, w, V):
    m = A.shape[0]
    _lib.call("gcg_syev", ctx.h, m, _p(A), _ld(A), _p(w), _p(V), _ld(V))
    return w, V


def syev_range(ctx, A, il, iu, w, V):
    """Eigenpairs il..iu (1-based inclusive) of symmetric A (gcg_syev_range)."""
    m = A.shape[0]
    _lib.call("gcg_syev_range", ctx.h, m, _p(A), _ld(A), int(il), int(iu), _p(w), _p(V), _ld(V))
    return w, V


def dgemm(ctx, A, B, Cm, ta=False, tb=False, alpha=1.0, beta=0.0):
    M = A.shape[1] if ta else A.shape[0]
    K = A.shape[0] if ta else A.shape[1]
    N = B.shape[0] if tb else B.shape[1]
    if Cm.shape != (M, N):
        raise InvalidShape(f"dgemm out {tuple(Cm.shape)} != {(M, N)}")
    _lib.call("gcg_dgemm", ctx.h, int(ta), int(tb), M, N, K, float(alpha), _p(A), _ld(A), _p(B),
              _ld(B), float(beta), _p(Cm), _ld(Cm))
    return Cm


def build_p(ctx, coeffs, num_x_rows, group_start, group_width, dep_tol):
    """solver._build_p on one device (gcg_build_p): the momentum coefficients (m x kept) or None."""
    m, d = coeffs.shape
    phat = ctx.empty(m, group_width)
    kept = C.c_int64(0)
    _lib.call("gcg_build_p", ctx.h, m, d, _p(coeffs), _ld(coeffs), int(num_x_rows),
              int(group_start), int(group_width), float(dep_tol), _p(phat), _ld(phat),
              C.byref(kept))
    k = int(kept.value)
    return phat[:, :k] if k > 0 else None


def symmetrize(ctx, A):
    _lib.call("gcg_symmetrize", ctx.h, A.shape[0], _p(A), _ld(A))
    return A


def svqb_prepare(ctx, G, dep_tol, Q, status, skip_tol=-1.0):
    w = G.shape[0]
    _lib.call("gcg_svqb_prepare", ctx.h, w, _p(G), _ld(G), float(dep_tol), float(skip_tol), _p(Q),
              _ld(Q), _p(status))


def deflate_status(ctx, R, dnew, dgks, status):
    """dnew may be a strided 1-D view (e.g. the diagonal of a Gram block)."""
    K, w = R.shape
    _lib.call("gcg_deflate_status", ctx.h, K, w, _p(R), _ld(R), _p(dnew), dnew.stride(0),
              float(dgks), _p(status))


def abar_assemble(ctx, d, lam, Pc, cross, Abar):
    np_ = 0 if Pc is None else Pc.shape[0]
    nw = 0 if cross is None else cross.shape[1]
    _lib.call("gcg_abar_assemble", ctx.h, d, np_, nw, _p(lam), _p(Pc), _ld(Pc), _p(cross),
              _ld(cross), _p(Abar), _ld(Abar))
    return Abar


def max_abs_diff(ctx, A, B, out):
    m, n = A.shape
    _lib.call("gcg_max_abs_diff", ctx.h, m, n, _p(A), _ld(A), _p(B), _ld(B), _p(out))
    return out


def count_le(ctx, vals, rel, out):
    _lib.call("gcg_count_le", ctx.h, vals.shape[0], _p(vals), float(rel), _p(out))


def scale_rsqrt(ctx, V, w, off, out):
    m = V.shape[0]
    _lib.call("gcg_scale_rsqrt", ctx.h, m, int(off), _p(V), _ld(V), _p(w), _p(out), _ld(out))
    return out


def ritz_residuals(ctx, AX, X, BX, lam, mode, out):
    n, k = X.shape
    _lib.call("gcg_ritz_residuals", ctx.h, n, k, _p(AX), _ld(AX), _p(X), _ld(X), _p(BX), _ld(BX),
              _p(lam), int(mode), _p(out))
    return out


def fp64_peak(ctx, mode="dmma", iters=4096, reps=5):
    """Measured FP64 throughput (TFLOP/s) of DMMA.8x8x4 ('dmma') or DFMA ('dfma') chains."""
    sink = ctx.empty(1)
    flops = C.c_double()
    m = 1 if mode == "dmma" else 0
    _lib.call("gcg_fp64_peak", ctx.h, m, int(iters), C.byref(flops), _p(sink))  # warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(reps):
        e0.record(ctx.stream)
        _lib.call("gcg_fp64_peak", ctx.h, m, int(iters), C.byref(flops), _p(sink))
        e1.record(ctx.stream)
        e1.synchronize()
        best = max(best, flops.value / (e0.elapsed_time(e1) / 1e3) / 1e12)
    return best


def gather_rows(ctx, idx, X, out):
    """out[i, :] = X[idx[i], :] (idx int32 on device)."""
    k = X.shape[1]
    _lib.call("gcg_gather_rows", ctx.h, idx.shape[0], _p(idx), k, _p(X), _ld(X), _p(out), _ld(out))
    return out


def ritz_sums(ctx, AX, X, BX, lam, mode, sums):
    n, k = X.shape
    _lib.call("gcg_ritz_sums", ctx.h, n, k, _p(AX), _ld(AX), _p(X), _ld(X), _p(BX), _ld(BX),
              _p(lam), int(mode), _p(sums))
    return sums


def ritz_finish(ctx, sums, lam, mode, out):
    _lib.call("gcg_ritz_finish", ctx.h, out.shape[0], _p(sums), _p(lam), int(mode), _p(out))
    return out


def block_cg_dist(ctx, A, vals, shift, rhs, x, max_iters, rel_tol, sweeps, conv, frozen, relres,
                  dist):
    n, k = rhs.shape
    _lib.call("gcg_block_cg_dist", ctx.h, n, A.nnz, _p(A.rowptr), _p(A.colidx), _p(vals),
              float(shift), k, _p(rhs), _ld(rhs), _p(x), _ld(x), int(max_iters), float(rel_tol),
              _p(sweeps), _p(conv), _p(frozen), _p(relres), C.byref(dist))


def block_cg(ctx, A, vals, shift, rhs, x, max_iters, rel_tol, sweeps, conv, frozen, relres,
             x0=None):
    n, k = x.shape
    if x0 is not None:
        if x0.shape != x.shape:
            raise InvalidShape(f"x0 {tuple(x0.shape)} != x {tuple(x.shape)}")
        _lib.call("gcg_block_cg_x0", ctx.h, n, A.nnz, _p(A.rowptr), _p(A.colidx), _p(vals),
                  float(shift), k, _p(rhs), _ld(rhs), _p(x0), _ld(x0), _p(x), _ld(x),
                  int(max_iters), float(rel_tol), _p(sweeps), _p(conv), _p(frozen), _p(relres))
        return
    _lib.call("gcg_block_cg", ctx.h, n, A.nnz, _p(A.rowptr), _p(A.colidx), _p(vals), float(shift), k,
              _p(rhs), _ld(rhs), _p(x), _ld(x), int(max_iters), float(rel_tol), _p(sweeps),
              _p(conv), _p(frozen), _p(relres))


def col_scale_copy(ctx, s, X, Y):
    """Y = X diag(s) in one pass (gcg_col_scale_copy)."""
    n, k = X.shape
    _lib.call("gcg_col_scale_copy", ctx.h, n, k, _p(s), _p(X), _ld(X), _p(Y), _ld(Y))
    return Y


def fill_normal(ctx, X, row0, seed):
    """X[i, c] = seeded N(0,1) of global row row0 + i (Philox, gcg_fill_normal)."""
    n, k = X.shape
    _lib.call("gcg_fill_normal", ctx.h, n, k, int(row0), int(seed) & (2**64 - 1), _p(X), _ld(X))
    return X


def csr_check(ctx, A):
    """(max |a|, max |a - a'|, #non-finite, #bad columns) of a square DeviceCsr (gcg_csr_check)."""
    out = (C.c_double * 4)()
    _lib.call("gcg_csr_check", ctx.h, A.n, _p(A.rowptr), _p(A.colidx), _p(A.val), out)
    return float(out[0]), float(out[1]), int(out[2]), int(out[3])
