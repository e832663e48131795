"""Small dense symmetric eigenproblems on device (no CPU fallback).

Reference: dense.py:63-133 — `sym_eig_full`, `sym_eig_range` (1-based inclusive
index range, optional split over workers), `gram_svd`; eigenvalues ascending,
eigenvector signs fixed so the largest-magnitude entry is positive (first
index on ties).

Device matrices are row-major float64 tensors.  Full spectra of orders <= 64
run the one-CTA Jacobi kernel; orders 65..1024 (every BASELINE Rayleigh-Ritz
order, up to cfg5's 1000) and every index range run csrc/eig.cu: Householder
tridiagonalisation (one CTA up to 224, multi-CTA above), bisection of the
requested indices, inverse iteration, back-transformation — no cuSOLVER
(``_lib.cusolver_calls()`` counts the calls beyond 1024).  The split-range solve of the paper's
parallel Rayleigh-Ritz is ``sym_eig_range(..., workers=w)``
on one device, and ``sym_eig_range_split`` across the ranks of a distributed
solve (each rank one slice, then an ordered all-gather).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import device as D
from .errors import InvalidRange, InvalidShape

__all__ = ["SpectralDecomposition", "sym_eig_full", "sym_eig_range", "sym_eig_range_split",
           "gram_svd", "split_ranges"]

_MIN_PAIRS_PER_WORKER = 10  # dense.py:33


@dataclass
class SpectralDecomposition:
    """values (m,) ascending and vectors (m, k) as device tensors."""

    values: torch.Tensor
    vectors: torch.Tensor


def _check_square(m):
    if m.dim() != 2 or m.shape[0] != m.shape[1]:
        raise InvalidShape(f"matrix must be square 2-D, got shape {tuple(m.shape)}")
    return m.shape[0]


def sym_eig_full(ctx, m, symmetrize=False):
    """All eigenpairs of the symmetric device matrix ``m`` (dense.py:74-82)."""
    n = _check_square(m)
    if symmetrize:
        m = m.clone()
        D.symmetrize(ctx, m)
    w = ctx.empty(n)
    # even row stride: coefficient blocks sliced from it stay 16-byte aligned row by
    # row, which the bulk-staged LinComb needs
    v = ctx.empty(n, n + (n & 1))[:, :n]
    D.syev(ctx, m, w, v)
    return SpectralDecomposition(w, v)


def split_ranges(lo, hi, workers):
    """Slices of lo..hi (1-based inclusive), each >= 10 pairs (dense.py:105-108)."""
    npairs = hi - lo + 1
    nw = min(int(workers), npairs // _MIN_PAIRS_PER_WORKER)
    if nw <= 1:
        return [(lo, hi)]
    cuts = np.linspace(lo - 1, hi, nw + 1).astype(int)
    return [(int(a) + 1, int(b)) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]


def _range_into(ctx, m, a, b, w, v):
    D.syev_range(ctx, m, a, b, w, v)


def sym_eig_range(ctx, m, lo, hi, workers=1):
    """Eigenpairs lo..hi (1-based inclusive) of a symmetric device matrix (dense.py:93-117).

    ``workers > 1`` computes the index range in slices of >= 10 pairs and
    concatenates them, as the reference's threaded path; like the reference,
    eigenvectors of a degenerate cluster straddling a slice boundary are not
    guaranteed mutually orthogonal — the single-slice path is the reference."""
    n = _check_square(m)
    if not (1 <= lo <= hi <= n):
        raise InvalidRange(f"range {lo}..{hi} invalid for dimension {n}")
    k = hi - lo + 1
    w = ctx.empty(k)
    v = ctx.empty(n, k)
    for a, b in split_ranges(lo, hi, workers):
        _range_into(ctx, m, a, b, w[a - lo:b - lo + 1], v[:, a - lo:b - lo + 1])
    return SpectralDecomposition(w, v)


def sym_eig_range_split(ops, m, lo, hi):
    """Split-range RR across the ranks of a distributed solve:
    rank r computes slice r of lo..hi (>= 10 pairs per slice; ranks beyond the
    slice count idle) and the slices are concatenated by an ordered all-gather,
    so every rank holds the identical full result."""
    n = _check_square(m)
    if not (1 <= lo <= hi <= n):
        raise InvalidRange(f"range {lo}..{hi} invalid for dimension {n}")
    dev = ops.dev
    k = hi - lo + 1
    ranges = split_ranges(lo, hi, ops.size)
    # one slab per rank, [values | vectors^T] so the gather is a single buffer
    out = dev.zeros(k, n + 1)
    if ops.rank < len(ranges):
        a, b = ranges[ops.rank]
        kk = b - a + 1
        w = dev.empty(kk)
        v = dev.empty(n, kk)
        D.syev_range(dev, m, a, b, w, v)
        out[a - lo:b - lo + 1, 0] = w
        out[a - lo:b - lo + 1, 1:] = v.t()
    ops.allgather_sum_small(out)  # disjoint slices: the ordered sum is a concatenation
    return SpectralDecomposition(out[:, 0].contiguous(), out[:, 1:].t().contiguous())


def gram_svd(ctx, m):
    """Spectral factorisation of a symmetric PSD Gram block (dense.py:120-133)."""
    return sym_eig_full(ctx, m)
