"""Device-resident sparse operators (MatDotMultiVec).

Reference: CsrOperator (operators.py:75-114), ShiftedOperator (operators.py:136-165),
as_operator (operators.py:168-179).

B200 layout: CSR with int32 row pointers / column indices and fp64 values in
HBM.  For a generalized problem A and B are stored on ONE shared pattern (the
union of their patterns, explicit zeros kept), so the damped operator
A - theta*B used by every CG sweep is a single value stream
S = A.val - theta*B.val (one nnz-length axpby per shift change) and the SpMM
reads one index stream instead of two.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse

from . import _lib
from . import device as D
from .errors import InvalidMatrix, InvalidShape

__all__ = ["DeviceCsr", "DeviceSell", "DeviceProblem", "as_device_problem", "validate_symmetric",
           "validate_device"]

_SYM_RTOL = 1e-12  # operators.py:26


def validate_symmetric(sp, name="operator"):
    """Reference validation (operators.py:79-87): square, finite, symmetric to 1e-12*scale."""
    if sp.shape[0] != sp.shape[1]:
        raise InvalidShape(f"sparse {name} must be square, got {sp.shape}")
    if not np.isfinite(sp.data).all():
        raise InvalidMatrix(f"sparse {name} has non-finite entries")
    defect = abs(sp - sp.T)
    scale = max(1.0, float(np.abs(sp.data).max(initial=0.0)))
    if defect.nnz and defect.max() > _SYM_RTOL * scale:
        raise InvalidMatrix(f"sparse {name} is not symmetric")


class DeviceCsr:
    """A CSR matrix in HBM: rowptr (n+1, int32), colidx (nnz, int32), val (nnz, f64)."""

    kind = "csr-sparse"

    def __init__(self, ctx, rowptr, colidx, val, n):
        self.ctx = ctx
        self.rowptr, self.colidx, self.val = rowptr, colidx, val
        self.n = self.dim = int(n)

    @property
    def nnz(self):
        return int(self.colidx.shape[0])

    @classmethod
    def from_scipy(cls, ctx, sp, values=None):
        sp = scipy.sparse.csr_matrix(sp)
        if sp.nnz >= 2**31 or sp.shape[0] >= 2**31:
            raise InvalidShape("CSR too large for int32 indices")
        # np.asarray: no host copy when the arrays already have the device dtypes (so
        # arrays in page-locked memory go straight to a DMA)
        rp = ctx.upload(np.asarray(sp.indptr, dtype=np.int32))
        ci = ctx.upload(np.asarray(sp.indices, dtype=np.int32))
        v = ctx.upload(np.asarray(sp.data if values is None else values, dtype=np.float64))
        return cls(ctx, rp, ci, v, sp.shape[0])

    def with_values(self, val):
        return DeviceCsr(self.ctx, self.rowptr, self.colidx, val, self.n)

    def apply(self, x, out, **kw):
        """out = A @ x (row-major device multivectors); kw forwards the fused epilogue."""
        return D.spmm(self.ctx, self, x, out, **kw)

    def bytes_per_apply(self, k):
        """Algorithmic HBM bytes of one SpMM with k columns."""
        return 12 * self.nnz + 4 * (self.n + 1) + 16 * self.n * k


class DeviceSell:
    """SELL-C-sigma copy of a DeviceCsr (C = 32, rows length-sorted in windows of 1024
    unless sigma=1): built on the device (gcg_sell_size / gcg_csr_to_sell), applied by
    gcg_spmm_sell with the CSR kernel's epilogues and the same results.  MatDotMultiVec
    on the sliced-ELLPACK format of SURVEY §8(b); the solver's block CG keeps CSR."""

    kind = "sell-sparse"

    def __init__(self, csr, sigma=1024):
        import ctypes as C
        import torch

        ctx = csr.ctx
        self.ctx, self.n, self.dim, self.nnz = ctx, csr.n, csr.n, csr.nnz
        ns, nz = C.c_int64(0), C.c_int64(0)
        _lib.call("gcg_sell_size", ctx.h, csr.n, D._p(csr.rowptr), int(sigma), C.byref(ns),
                  C.byref(nz))
        self.nslices, self.nnz_padded = int(ns.value), int(nz.value)
        self.slice_ptr = ctx.empty(self.nslices + 1, dtype=torch.int64)
        self.perm = ctx.empty(csr.n, dtype=torch.int32)
        self.col = ctx.empty(max(self.nnz_padded, 1), dtype=torch.int32)
        self.val = ctx.empty(max(self.nnz_padded, 1))
        _lib.call("gcg_csr_to_sell", ctx.h, csr.n, D._p(csr.rowptr), D._p(csr.colidx),
                  D._p(csr.val), int(sigma), D._p(self.slice_ptr), D._p(self.perm),
                  D._p(self.col), D._p(self.val))

    def apply(self, x, out, alpha=1.0, gamma=0.0, Z=None, beta=0.0, Yin=None, dot_mode=0, W=None,
              dots=None):
        n, k = out.shape
        if x.shape != out.shape or n != self.n:
            raise InvalidShape(f"sell apply: X {tuple(x.shape)} / Y {tuple(out.shape)} vs dim {self.n}")
        _lib.call("gcg_spmm_sell", self.ctx.h, n, self.nslices, D._p(self.slice_ptr),
                  D._p(self.perm), D._p(self.col), D._p(self.val), k, D._p(x), D._ld(x),
                  float(alpha), float(gamma), D._p(Z), D._ld(Z), float(beta), D._p(Yin),
                  D._ld(Yin), D._p(out), D._ld(out), int(dot_mode), D._p(W), D._ld(W),
                  D._p(dots))
        return out


class DeviceProblem:
    """A (and optionally B) on one shared CSR pattern, plus the shifted-value buffer."""

    def __init__(self, ctx, a, b=None):
        self.ctx = ctx
        if b is not None:
            a, b = _shared_pattern(a, b)
        self.A = DeviceCsr.from_scipy(ctx, a)
        self.B = None
        if b is not None:
            self.B = self.A.with_values(ctx.upload(b.data.astype(np.float64)))
        self.n = self.A.n
        self._shift_vals = None
        self._shift_theta = None

    @classmethod
    def from_device(cls, ctx, A, B=None):
        """Wrap operators already in HBM (e.g. assembled by devgen); B must share A's pattern."""
        self = cls.__new__(cls)
        self.ctx = ctx
        self.A = A
        self.B = B
        self.n = A.n
        self._shift_vals = None
        self._shift_theta = None
        return self

    def shifted(self, theta):
        """(values, diag_shift) such that op = CSR(values) + diag_shift*I equals A - theta*B."""
        if theta == 0.0:
            return self.A.val, 0.0
        if self.B is None:
            return self.A.val, -float(theta)
        if self._shift_theta != theta:
            if self._shift_vals is None:
                self._shift_vals = self.ctx.empty(self.A.nnz)
            s = self._shift_vals.view(-1, 1)
            D.copy(self.ctx, self.A.val.view(-1, 1), s)
            D.axpby(self.ctx, -float(theta), self.B.val.view(-1, 1), 1.0, s)
            self._shift_theta = theta
        return self._shift_vals, 0.0


def _shared_pattern(a, b):
    """Return (a, b) as CSR matrices on the union of their sparsity patterns."""
    a = scipy.sparse.csr_matrix(a, dtype=np.float64)
    b = scipy.sparse.csr_matrix(b, dtype=np.float64)
    a.sum_duplicates()
    b.sum_duplicates()
    a.sort_indices()
    b.sort_indices()
    if a.shape == b.shape and np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices):
        return a, b
    pat = (abs(a) + abs(b)).tocsr()
    pat.data[:] = 1.0
    pat.sort_indices()
    au = _on_pattern(a, pat)
    bu = _on_pattern(b, pat)
    return au, bu


def _on_pattern(m, pat):
    """Values of m scattered onto pattern `pat` (explicit zeros where m has none)."""
    out = pat.copy().astype(np.float64)
    out.data[:] = 0.0
    coo = m.tocoo()
    n = np.int64(pat.shape[1])
    # canonical CSR keys row*n + col are globally sorted, so one searchsorted places them
    rows = np.repeat(np.arange(pat.shape[0], dtype=np.int64), np.diff(pat.indptr))
    keys = rows * n + pat.indices.astype(np.int64)
    pos = np.searchsorted(keys, coo.row.astype(np.int64) * n + coo.col.astype(np.int64))
    np.add.at(out.data, pos, coo.data)
    return out


def as_device_problem(ctx, a, b=None, validate=True):
    """Coerce host matrices to a DeviceProblem (reference: as_operator, operators.py:168-179).

    Accepts scipy sparse matrices or dense 2-D arrays (converted to CSR).
    """
    def coerce(m, name):
        if scipy.sparse.issparse(m):
            sp = scipy.sparse.csr_matrix(m, dtype=np.float64)
        else:
            arr = np.asarray(m, dtype=np.float64)
            if arr.ndim == 1:
                sp = scipy.sparse.diags(arr, format="csr")
            elif arr.ndim == 2:
                sp = scipy.sparse.csr_matrix(arr)
            else:
                raise InvalidShape(f"cannot build an operator from shape {arr.shape}")
        sp.sum_duplicates()
        if sp.shape[0] != sp.shape[1]:
            raise InvalidShape(f"sparse {name} must be square, got {sp.shape}")
        return sp

    sa = coerce(a, "A")
    sb = coerce(b, "B") if b is not None else None
    if sb is not None and sb.shape[0] != sa.shape[0]:
        raise InvalidShape(f"B dim {sb.shape[0]} != A dim {sa.shape[0]}")
    prob = DeviceProblem(ctx, sa, sb)
    if validate:
        # the reference's operator checks (operators.py:79-87) on the device copy
        for name, op in (("A", prob.A), ("B", prob.B)):
            if op is not None:
                validate_device(ctx, op, name)
    return prob


def validate_device(ctx, op, name="operator"):
    """Finite and symmetric to 1e-12 * max(1, max |a|) (operators.py:79-87), checked by
    gcg_csr_check on the matrix in HBM."""
    amax, defect, nonfinite, badcol = D.csr_check(ctx, op)
    if badcol:
        raise InvalidShape(f"sparse {name} has column indices outside 0..{op.n - 1}")
    if nonfinite:
        raise InvalidMatrix(f"sparse {name} has non-finite entries")
    if defect > _SYM_RTOL * max(1.0, amax):
        raise InvalidMatrix(f"sparse {name} is not symmetric")
