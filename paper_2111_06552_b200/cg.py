"""Block CG on device (GCG STEP 6: damped inverse power).

Reference: block_cg (cg.py:33-99), CgReport (cg.py:21-26).  The whole solve —
initial residual, up to ``max_iters`` sweeps, per-column stopping and
freezing — is enqueued by one C-ABI call (gcg_block_cg) without a host sync;
the report's fields are device tensors that are read back lazily.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import device as D
from .errors import InvalidShape

__all__ = ["CgReport", "block_cg"]


@dataclass
class CgReport:
    """Lazy mirror of cg.CgReport: fields resolve (one D2H) on first access."""

    _sweeps: torch.Tensor
    _conv: torch.Tensor
    _frozen: torch.Tensor
    _relres: torch.Tensor

    @property
    def iterations(self):
        return int(self._sweeps.item())

    @property
    def converged(self):
        return self._conv.cpu().numpy().astype(bool)

    @property
    def frozen(self):
        return self._frozen.cpu().numpy().astype(bool)

    @property
    def relative_residuals(self):
        return self._relres.cpu().numpy()


def block_cg(ctx, problem, theta, rhs, x, max_iters=30, rel_tol=0.01):
    """Solve (A - theta*B) x = rhs from the initial guess already in ``x`` (updated in place).

    ``rhs`` and ``x`` are row-major device multivectors (n x k views).
    """
    if rhs.shape != x.shape:
        raise InvalidShape(f"x0 shape {tuple(x.shape)} != rhs shape {tuple(rhs.shape)}")
    if rhs.shape[0] != problem.n:
        raise InvalidShape(f"operator dim {problem.n} != rhs dim {rhs.shape[0]}")
    k = rhs.shape[1]
    sweeps = ctx.zeros(1, dtype=torch.int32)
    conv = ctx.zeros(k, dtype=torch.int8)
    frozen = ctx.zeros(k, dtype=torch.int8)
    relres = ctx.zeros(k)
    vals, shift = problem.shifted(theta)
    D.block_cg(ctx, problem.A, vals, shift, rhs, x, max_iters, rel_tol, sweeps, conv, frozen, relres)
    return x, CgReport(sweeps, conv, frozen, relres)
