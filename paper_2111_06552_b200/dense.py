"""Small dense symmetric eigenproblems on device (no CPU fallback).

Reference: dense.py:63-133 — `sym_eig_full`, `sym_eig_range` (1-based inclusive
index range), `gram_svd`; eigenvalues ascending, eigenvector signs fixed so
the largest-magnitude entry is positive (first index on ties).

Device matrices are row-major float64 tensors.  Orders <= 64 run the one-CTA
Jacobi kernel, larger ones cuSOLVER syevd (see csrc/dense.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import device as D
from .errors import InvalidRange, InvalidShape

__all__ = ["SpectralDecomposition", "sym_eig_full", "sym_eig_range", "gram_svd"]


@dataclass
class SpectralDecomposition:
    """values (m,) ascending and vectors (m, k) as device tensors."""

    values: torch.Tensor
    vectors: torch.Tensor


def sym_eig_full(ctx, m, symmetrize=False):
    """All eigenpairs of the symmetric device matrix ``m`` (dense.py:74-82)."""
    if m.dim() != 2 or m.shape[0] != m.shape[1]:
        raise InvalidShape(f"matrix must be square 2-D, got shape {tuple(m.shape)}")
    n = m.shape[0]
    if symmetrize:
        m = m.clone()
        D.symmetrize(ctx, m)
    w = ctx.empty(n)
    v = ctx.empty(n, n)
    D.syev(ctx, m, w, v)
    return SpectralDecomposition(w, v)


def sym_eig_range(ctx, m, lo, hi):
    """Eigenpairs lo..hi (1-based inclusive) of a symmetric device matrix (dense.py:93-117)."""
    n = m.shape[0]
    if not (1 <= lo <= hi <= n):
        raise InvalidRange(f"range {lo}..{hi} invalid for dimension {n}")
    full = sym_eig_full(ctx, m)
    return SpectralDecomposition(full.values[lo - 1:hi], full.vectors[:, lo - 1:hi])


def gram_svd(ctx, m):
    """Spectral factorisation of a symmetric PSD Gram block (dense.py:120-133)."""
    return sym_eig_full(ctx, m)
