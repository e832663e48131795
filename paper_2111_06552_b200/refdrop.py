"""Drop the B200 path into the reference package (`gcgeig`) — the reference-side plugin.

Three levels, each replacing one reference interface and keeping its signature,
argument meaning and error classes:

1. kernels: the `sm100` backend of the reference's registry (refbackend.py,
   _kernels/__init__.py:11-63) — csr_matvec / inner_product / axpby;
2. operators: :func:`csr_operator` returns an ``Sm100CsrOperator``, a subclass of
   the reference's ``CsrOperator`` (operators.py:75-114) whose matrix stays in HBM
   (gcgeig_csr_create) and whose ``apply`` runs the B200 SpMM (gcgeig_csr_apply).
   The reference's ``as_operator`` passes it through unchanged (operators.py:168-170),
   so the reference's own GCG driver then does every A*X / B*X product on the GPU.
   (The stock ``CsrOperator.apply`` only calls ``kernels.csr_matvec`` when the
   backend is named "compiled", operators.py:105 — with `sm100` selected it would
   still multiply in scipy.)
3. driver: :func:`gcg_solve`, :func:`recursive_orth_svd`, :func:`orth_against`,
   :func:`modified_block_orth` take the reference's host arguments (F-order numpy
   blocks updated in place, reference ``SolverConfig`` / ``OrthConfig``, reference
   operator objects) and run the whole device path of this package; results come
   back as the reference's own dataclasses and errors as the reference's classes.

``install(gcgeig)`` does all three: registers the backend and rebinds the
package-level entry points (gcgeig.gcg_solve, gcgeig.solver.gcg_solve, the orth
functions), so code and tests written against the reference run on the B200
unchanged (tests/test_gpu_refdrop.py runs the reference's own test files this way).
"""

from __future__ import annotations

import ctypes as C
import sys

import numpy as np
import scipy.sparse

from . import _lib
from . import errors as E

__all__ = ["csr_operator", "gcg_solve", "recursive_orth_svd", "orth_against",
           "modified_block_orth", "install"]

_DENSE_MATERIALIZE_MAX = 4096  # generic matrix-free operators are materialised up to this n


def _ref():
    return sys.modules.get("gcgeig") or __import__("gcgeig")


def _ref_error(exc):
    """The reference's exception class of the same name (errors.py:4-47)."""
    cls = getattr(_ref().errors, type(exc).__name__, None)
    if cls is None or not isinstance(exc, E.GcgError):
        return exc
    return cls(str(exc))


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else C.c_void_p(0)


# ---- level 2: the operator ------------------------------------------------------------

_OP_CLASS = None


def _operator_class():
    global _OP_CLASS
    if _OP_CLASS is not None:
        return _OP_CLASS
    base = _ref().operators.CsrOperator

    class Sm100CsrOperator(base):
        """CsrOperator whose matrix lives in HBM and whose apply is the B200 SpMM."""

        def __init__(self, matrix):
            super().__init__(matrix)  # the reference's validation (operators.py:79-96)
            h = C.c_void_p()
            _lib.check(_lib.load().gcgeig_csr_create(
                _p(self.indptr), _p(self.indices), _p(self.data), self.dim, self.dim,
                C.byref(h)), "gcgeig_csr_create")
            self._handle = h

        def apply(self, x, out=None):
            out = self._out(x, out)
            k = x.shape[1]
            if k == 0:
                return out
            xs = x if (x.dtype == np.float64 and x.flags.f_contiguous) else \
                np.asfortranarray(x, dtype=np.float64)
            tgt = out if out.flags.f_contiguous else np.empty(out.shape, order="F")
            _lib.check(_lib.load().gcgeig_csr_apply(self._handle, _p(xs), k, max(self.dim, 1),
                                                    _p(tgt), max(self.dim, 1)),
                       "gcgeig_csr_apply")
            if tgt is not out:
                out[...] = tgt
            return out

        def __del__(self):  # pragma: no cover
            h = getattr(self, "_handle", None)
            if h is not None and h.value:
                try:
                    _lib.load().gcgeig_csr_destroy(h)
                except Exception:
                    pass
                self._handle = None

    _OP_CLASS = Sm100CsrOperator
    return _OP_CLASS


def csr_operator(matrix):
    """A reference ``CsrOperator`` (subclass) with the matrix resident in HBM."""
    return _operator_class()(matrix)


# ---- level 3: the driver ---------------------------------------------------------------


def _host_matrix(obj):
    """Reference operator / scipy / ndarray -> what this package's gcg_solve accepts."""
    if obj is None or scipy.sparse.issparse(obj) or isinstance(obj, np.ndarray):
        return obj
    ops = _ref().operators
    if isinstance(obj, ops.CsrOperator):
        return obj.tocsr()
    if isinstance(obj, ops.DenseOperator):
        return obj.a
    if isinstance(obj, ops.DiagonalOperator):
        return scipy.sparse.diags(obj.d, format="csr")
    if isinstance(obj, ops.LinearOperator):
        # a matrix-free operator: materialise column blocks of the identity
        n = obj.dim
        if n > _DENSE_MATERIALIZE_MAX:
            raise _ref().errors.Unsupported(
                f"matrix-free {obj.kind} operator of dim {n} cannot be moved to the device")
        return np.asarray(obj.apply(np.asfortranarray(np.eye(n))))
    return np.asarray(obj)


def _orth_cfg(cfg):
    from .orth import OrthConfig

    if cfg is None:
        return OrthConfig()
    return OrthConfig(block_width=cfg.block_width, svd_leaf=cfg.svd_leaf,
                      reorth_tol=cfg.reorth_tol, dependence_tol=cfg.dependence_tol,
                      max_reorth_passes=cfg.max_reorth_passes)


def _solver_cfg(cfg):
    from .solver import SolverConfig

    if cfg is None:
        return SolverConfig()
    fields = ("num_eigen", "tol", "block_size", "size_x", "max_gcg_iters", "cg_max_iters",
              "cg_rel_tol", "shift_mode", "moving", "seed", "deterministic", "collect_history",
              "stall_window", "instrument_orth", "cross_check_abar")
    return SolverConfig(**{f: getattr(cfg, f) for f in fields}, orth=_orth_cfg(cfg.orth))


def gcg_solve(a, b=None, config=None):
    """Reference signature (solver.py:226): host inputs, reference SolverReport out."""
    from . import solver as S

    R = _ref()
    try:
        rep = S.gcg_solve(_host_matrix(a), _host_matrix(b), _solver_cfg(config))
    except E.GcgError as exc:
        raise _ref_error(exc) from exc
    hist = [R.solver.IterationRecord(h.iteration, h.num_converged, h.first_unconverged_residual,
                                     h.theta, h.cg_iterations, h.basis_size, h.orth_reductions,
                                     dict(h.timings), h.basis_defect, h.abar_defect)
            for h in rep.history]
    return R.solver.SolverReport(rep.status, rep.eigenvalues, rep.eigenvectors,
                                 rep.num_converged, rep.iterations, rep.residuals, hist,
                                 rep.stagnated, rep.max_projection_dim, rep.total_reductions,
                                 rep.backend)


def _device_block(x):
    import torch

    from . import device as D

    dev = D.default_context()
    return dev, torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev.device)


def _writeback(dst, src):
    dst[...] = src.cpu().numpy()


def _device_b(dev, b):
    if b is None:
        return None
    from .operators import DeviceCsr

    m = _host_matrix(b)
    return DeviceCsr.from_scipy(dev, scipy.sparse.csr_matrix(m))


def _outcome(o):
    return _ref().orth.OrthOutcome(o.num_kept, list(o.replaced_indices), o.reduction_count)


def _orth_call(fn, x, *args, b=None, cfg=None, **kw):
    dev, xd = _device_block(x)
    try:
        out = fn(dev, xd, *args, b=_device_b(dev, b), cfg=_orth_cfg(cfg), **kw)
    except E.GcgError as exc:
        _writeback(x, xd)
        raise _ref_error(exc) from exc
    _writeback(x, xd)
    return _outcome(out)


def recursive_orth_svd(x, s=None, e=None, b=None, cfg=None):
    """orth.recursive_orth_svd (orth.py:207-226) on an F-order host block, in place."""
    from . import orth as O

    return _orth_call(O.recursive_orth_svd, x, s, e, b=b, cfg=cfg)


def orth_against(x, basis, b=None, cfg=None):
    """orth.orth_against (orth.py:339-372) on F-order host blocks, x in place."""
    from . import orth as O

    basis_d = None
    if basis is not None:
        _, basis_d = _device_block(basis)
    return _orth_call(O.orth_against, x, basis_d, b=b, cfg=cfg)


def modified_block_orth(x, x0=None, b=None, cfg=None):
    """orth.modified_block_orth (orth.py:304-336, Alg. 2) on F-order host blocks."""
    from . import orth as O

    x0_d = None
    if x0 is not None:
        _, x0_d = _device_block(x0)
    return _orth_call(O.modified_block_orth, x, b=b, cfg=cfg, x0=x0_d)


def install(gcgeig=None):
    """Register the `sm100` backend and rebind the reference's entry points to the B200
    path.  Returns the gcgeig module."""
    from . import refbackend

    R = gcgeig if gcgeig is not None else _ref()
    refbackend.register(R._kernels)
    R.gcg_solve = R.solver.gcg_solve = gcg_solve
    for name in ("recursive_orth_svd", "orth_against", "modified_block_orth"):
        fn = globals()[name]
        setattr(R, name, fn)
        setattr(R.orth, name, fn)
    R.sm100_csr_operator = csr_operator
    return R
