"""`sm100` kernel backend for the reference's backend registry.

Reference contract: a backend is any module with ``name`` and the three
functions of gcgeig/_kernels/_numpy_impl.py:12-47 / _cy.pyx:11-65 —
``csr_matvec(indptr, indices, data, x, out)``, ``inner_product(x, y, out,
chunk, deterministic)``, ``axpby(alpha, x, beta, y)`` on column-major host
arrays.  This module implements them through the host-buffer tier of the C
ABI (gcgeig_* in include/gcgb200.h): H2D, B200 kernel, D2H.

    import gcgeig._kernels as K
    from paper_2111_06552_b200 import refbackend
    refbackend.register(K)          # K.available_backends() now lists "sm100"
    K.use_backend("sm100")

The name is deliberately not "cuda": the reference test-suite asserts that
use_backend("cuda") raises (test_kernels.py:38-40).
"""

from __future__ import annotations

import ctypes as C
import sys

import numpy as np

from . import _lib

name = "sm100"


def _ptr(a):
    return C.c_void_p(a.ctypes.data)


def _colmajor(x):
    """(array, column stride in elements) for a 2-D float64 array with unit row stride."""
    if x.ndim != 2:
        raise ValueError("expected a 2-D block")
    if x.dtype != np.float64 or x.strides[0] != 8 or (x.shape[1] > 1 and x.strides[1] % 8):
        x = np.asfortranarray(x, dtype=np.float64)
    ld = x.strides[1] // 8 if x.shape[1] > 1 else max(x.shape[0], 1)
    return x, max(ld, x.shape[0], 1)


def csr_matvec(indptr, indices, data, x, out):
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    data = np.ascontiguousarray(data, dtype=np.float64)
    xs, ldx = _colmajor(x)
    nrow = indptr.shape[0] - 1
    if out.strides[0] == 8 and out.dtype == np.float64 and (out.shape[1] <= 1 or out.strides[1] % 8 == 0):
        tgt, ldo = out, (out.strides[1] // 8 if out.shape[1] > 1 else max(nrow, 1))
    else:
        tgt = np.empty((nrow, xs.shape[1]), order="F")
        ldo = max(nrow, 1)
    _lib.check(_lib.load().gcgeig_csr_matvec(_ptr(indptr), _ptr(indices), _ptr(data), nrow,
                                             xs.shape[0], _ptr(xs), xs.shape[1], ldx, _ptr(tgt),
                                             max(ldo, nrow, 1)), "gcgeig_csr_matvec")
    if tgt is not out:
        out[...] = tgt
    return out


def inner_product(x, y, out, chunk, deterministic):
    xs, ldx = _colmajor(x)
    ys, ldy = _colmajor(y)
    rs, cs = out.strides[0] // 8, out.strides[1] // 8
    if out.dtype != np.float64 or out.strides[0] % 8 or out.strides[1] % 8:
        raise ValueError("out must be a float64 view")
    _lib.check(_lib.load().gcgeig_inner_product(_ptr(xs), xs.shape[0], xs.shape[1], ldx, _ptr(ys),
                                                ys.shape[1], ldy, _ptr(out), rs, cs, int(chunk),
                                                int(bool(deterministic))), "gcgeig_inner_product")
    return out


def axpby(alpha, x, beta, y):
    xs, ldx = _colmajor(x)
    if y.dtype != np.float64 or y.strides[0] != 8:
        raise ValueError("y must be a column-major float64 block")
    ldy = y.strides[1] // 8 if y.shape[1] > 1 else max(y.shape[0], 1)
    _lib.check(_lib.load().gcgeig_axpby(float(alpha), _ptr(xs), xs.shape[0], xs.shape[1], ldx,
                                        float(beta), _ptr(y), max(ldy, y.shape[0], 1)),
               "gcgeig_axpby")
    return y


def register(kernels_module=None):
    """Insert this backend into gcgeig._kernels._IMPLS (the reference registry)."""
    if kernels_module is None:
        kernels_module = sys.modules["gcgeig._kernels"]
    kernels_module._IMPLS[name] = sys.modules[__name__]
    return name
