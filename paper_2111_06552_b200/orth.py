"""B-orthogonalisation on device: Alg. 3 (recursive SVD-based) and orth_against.

Reference: orth.py — `_deflate_against` (:124-152), `_leaf_svqb` (:155-188),
`_recurse_svd` (:191-204), `recursive_orth_svd` (:207-226), `orth_against`
(:339-372), `_Ctx.pull_rear` (:95-108), `OrthConfig` (:48-62),
`OrthOutcome` (:65-69).

The control flow (recursion, repeat-until tests, dependent-column
replacement, reduction counts) is the reference's, run on the host; every
long-vector operation is a device kernel and each repeat decision costs one
small device->host read of a fused status record:

  deflation pass = Gram [basis | target]' (B target) -> (coefficients, squared
                   norms) + LinComb target -= basis R + status (max|R|, DGKS flag)
  SVQB pass      = Gram block' B block + one-CTA Jacobi/SVQB kernel
                   (defect, #dependent, Q = V/sqrt(lambda)) + LinComb block <- block Q

When the target columns sit right after the basis in the same arena (always
the case inside the recursion and for W against [X | P]), the squared norms
ride along in the Gram as the diagonal of its bottom block, so one pass over
the data yields both — the fused reduction the reference counts as one.

The first argument is an ops object (mvops.LocalOps / distributed.DistOps) or
a plain device Context; in a row-partitioned run every "reduction" is one
ordered all-gather sum, exactly the unit the reference counts.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import device as D
from .errors import AllDependent, InvalidRange, InvalidShape
from .mvops import LocalOps

__all__ = ["OrthConfig", "OrthOutcome", "recursive_orth_svd", "orth_against"]

_DGKS_RATIO = 0.5  # orth.py:43


@dataclass
class OrthConfig:
    """Same fields and defaults as orth.OrthConfig (orth.py:48-62)."""

    block_width: int | None = None
    svd_leaf: int | None = None
    reorth_tol: float = 1e-10
    dependence_tol: float = 1e-10
    max_reorth_passes: int = 3


@dataclass
class OrthOutcome:
    num_kept: int
    replaced_indices: list = field(default_factory=list)
    reduction_count: int = 0


class _NoProblem:
    B = None
    n = None


def _as_ops(obj):
    if isinstance(obj, LocalOps):
        return obj
    return LocalOps(obj, _NoProblem())  # a bare Context: single-GPU ops, no operator needed


def _adjacent(left, right):
    """True when `right` starts exactly where `left` ends in the same row-major storage."""
    if left.shape[1] == 0 or right.shape[1] == 0:
        return False
    if left.stride() != right.stride() or left.untyped_storage().data_ptr() != \
            right.untyped_storage().data_ptr():
        return False
    return right.data_ptr() == left.data_ptr() + left.shape[1] * left.element_size()


def _span(left, width):
    """View of `width` columns starting at left's first column (same storage)."""
    return left.as_strided((left.shape[0], width), left.stride())


class _State:
    """Per-call bookkeeping (orth.py:72-108)."""

    def __init__(self, ops, x, b, cfg, start, end):
        self.ops = ops
        self.dev = ops.dev
        self.x = x
        self.b = b
        self.cfg = cfg
        self.start = start
        self.active_end = end
        self.reductions = 0
        self.replaced = []
        self.leaf_width = 16
        self.status = self.dev.empty(4)

    def bdot(self, y):
        return y if self.b is None else self.ops.apply(self.b, y)

    def read_status(self, count):
        """Host copy of the decision record (identical on every rank)."""
        return self.ops.broadcast(self.status)[:count].tolist()

    def pull_rear(self, slot):
        self.replaced.append(slot)
        if self.active_end - 1 > slot:
            self.active_end -= 1
            D.copy(self.dev, self.x[:, self.active_end:self.active_end + 1],
                   self.x[:, slot:slot + 1])
            return True
        self.active_end = slot
        return False


def _deflate_against(st, basis, lo, hi):
    """Repeat-until deflation of x[:, lo:hi] against a B-orthonormal basis (orth.py:124-152)."""
    cfg, dev, ops = st.cfg, st.dev, st.ops
    passes = 0
    while passes < cfg.max_reorth_passes:
        hi = min(hi, st.active_end)
        K = basis.shape[1]
        if lo >= hi or K == 0:
            return passes
        target = st.x[:, lo:hi]
        w = hi - lo
        bt = st.bdot(target)
        if _adjacent(basis, target):
            g = dev.empty(K + w, w)
            ops.gram(_span(basis, K + w), bt, g)
            coef, dnew = g[:K], g[K:].diagonal()
        else:
            coef = dev.empty(K, w)
            ops.gram(basis, bt, coef)
            dnew = dev.empty(w)
            ops.col_dots(target, bt, dnew)
        st.reductions += 1
        passes += 1
        D.lincomb(dev, basis, coef, target, alpha=-1.0, beta=1.0)
        D.deflate_status(dev, coef, dnew, _DGKS_RATIO, st.status)
        rmax, risky = st.read_status(2)
        if rmax <= cfg.reorth_tol:
            return passes
        if not risky:
            return passes
    return passes


def _leaf_svqb(st, lo, hi):
    """Orthonormalise x[:, lo:hi] by repeated scaled Gram factorisations (orth.py:155-188)."""
    cfg, dev, ops = st.cfg, st.dev, st.ops
    passes = 0
    while True:
        hi = min(hi, st.active_end)
        if lo >= hi:
            return
        w = hi - lo
        block = st.x[:, lo:hi]
        g = dev.empty(w, w)
        ops.gram(block, st.bdot(block), g)
        st.reductions += 1
        passes += 1
        q = dev.empty(w, w)
        D.svqb_prepare(dev, g, cfg.dependence_tol, q, st.status, skip_tol=cfg.reorth_tol)
        defect, nbad, _ = st.read_status(3)
        if defect <= cfg.reorth_tol:
            return
        ops.broadcast(q)
        bad = int(nbad)
        kept = w - bad
        if kept > 0:
            tmp = dev.empty(block.shape[0], kept)
            D.lincomb(dev, block, q[:, :kept], tmp)
            D.copy(dev, tmp, block[:, :kept])
        if bad == 0:
            if passes >= cfg.max_reorth_passes:
                return
            continue
        for slot in range(lo + kept, hi):
            if not st.pull_rear(slot):
                break
        passes = 0


def _recurse_svd(st, lo, hi):
    """orth.py:191-204."""
    hi = min(hi, st.active_end)
    if lo >= hi:
        return
    width = hi - lo
    if width <= st.leaf_width:
        _leaf_svqb(st, lo, hi)
        return
    mid = lo + width // 2
    _recurse_svd(st, lo, mid)
    mid = min(mid, st.active_end)
    if lo < mid < st.active_end:
        _deflate_against(st, st.x[:, lo:mid], mid, hi)
    _recurse_svd(st, mid, hi)


def recursive_orth_svd(ops, x, s=None, e=None, b=None, cfg=None):
    """B-orthonormalise columns s..e (1-based, inclusive) of device block ``x`` in place."""
    ops = _as_ops(ops)
    cfg = cfg if cfg is not None else OrthConfig()
    ncols = x.shape[1]
    s = 1 if s is None else s
    e = ncols if e is None else e
    if not (1 <= s <= e <= ncols):
        raise InvalidRange(f"column range {s}..{e} invalid for width {ncols}")
    lo, hi = s - 1, e
    st = _State(ops, x, b, cfg, lo, hi)
    st.leaf_width = cfg.svd_leaf if cfg.svd_leaf is not None else min(hi - lo, 16)
    if st.leaf_width < 1:
        raise InvalidShape(f"svd_leaf must be >= 1, got {st.leaf_width}")
    _recurse_svd(st, lo, hi)
    kept = st.active_end - lo
    if kept <= 0:
        raise AllDependent("every column in the block is linearly dependent")
    return OrthOutcome(kept, st.replaced, st.reductions)


def orth_against(ops, x, basis, b=None, cfg=None):
    """Deflate ``x`` against ``basis``, Alg. 3, then deflate + SVQB the kept block (orth.py:339-372)."""
    ops = _as_ops(ops)
    cfg = cfg if cfg is not None else OrthConfig()
    if x.shape[1] == 0:
        return OrthOutcome(0, [], 0)
    st = _State(ops, x, b, cfg, 0, x.shape[1])
    have_basis = basis is not None and basis.shape[1] > 0
    if have_basis:
        if basis.shape[0] != x.shape[0]:
            raise InvalidShape(f"basis dim {basis.shape[0]} != block dim {x.shape[0]}")
        _deflate_against(st, basis, 0, x.shape[1])
    inner = recursive_orth_svd(ops, x, 1, x.shape[1], b=b, cfg=cfg)
    kept = inner.num_kept
    replaced = list(inner.replaced_indices)
    extra = 0
    if have_basis and kept > 0:
        post = _State(ops, x, b, cfg, 0, kept)
        _deflate_against(post, basis, 0, kept)
        _leaf_svqb(post, 0, kept)
        kept = post.active_end
        replaced += post.replaced
        extra = post.reductions
        if kept <= 0:
            raise AllDependent("every column in the block is linearly dependent")
    return OrthOutcome(kept, replaced, st.reductions + inner.reduction_count + extra)
