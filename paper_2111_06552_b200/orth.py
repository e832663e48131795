"""B-orthogonalisation on device: Alg. 3 (recursive SVD-based), orth_against and
Alg. 2 (block modified Gram-Schmidt).

Reference: orth.py — `_deflate_against` (:124-152), `_leaf_svqb` (:155-188),
`_recurse_svd` (:191-204), `recursive_orth_svd` (:207-226), `orth_against`
(:339-372), `_Ctx.pull_rear` (:95-108), `OrthConfig` (:48-62),
`OrthOutcome` (:65-69); Alg. 2: `_seed_local_norms` (:114-119), `_mgs_block`
(:229-269), `_block_deflate` (:272-301), `modified_block_orth` (:304-336).

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

import ctypes as C
import os

import numpy as np
import torch

from . import _lib
from . import device as D
from .errors import AllDependent, InvalidRange, InvalidShape
from .mvops import LocalOps

__all__ = ["OrthConfig", "OrthOutcome", "modified_block_orth", "recursive_orth_svd", "orth_against"]

_DGKS_RATIO = 0.5  # orth.py:43
# one GPU: the Alg. 3 decision loop runs natively (gcg_orth_recursive /
# gcg_orth_against, csrc/orth.cu); the Python control flow below serves the
# row-partitioned path (collectives per reduction) and Alg. 2.
_NATIVE = os.environ.get("GCG_ORTH_NATIVE", "1") != "0"
_REPAIR_RATIO = 1e-8  # orth.py:45


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
        # Alg. 2 only: host copies of the tracked squared B-norms and the largest
        # one seen (orth.py:87-88); Alg. 3 never reads them, so it skips the reads
        self.track = False
        self.scale = 0.0
        self.d = np.full(x.shape[1], np.nan)

    def note_scale(self, vals):
        top = float(np.max(vals, initial=0.0))
        if top > self.scale:
            self.scale = top

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
            self.d[slot] = self.d[self.active_end]
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
        if st.track:
            lost = dev.empty(w)
            D.col_dots(dev, coef, coef, lost)  # coef is replicated: a local reduction
            rec = torch.cat([st.ops.broadcast(st.status)[:2], dnew, lost]).cpu().numpy()
            rmax, risky = float(rec[0]), rec[1]
            dn, ls = rec[2:2 + w], rec[2 + w:]
            st.note_scale(dn)
            st.d[lo:hi] = np.maximum(dn if rmax <= cfg.reorth_tol else dn - ls, 0.0)
        else:
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


def _native_ok(ops, b):
    return _NATIVE and type(ops) is LocalOps and (b is None or hasattr(b, "rowptr"))


def _native(name, ops, x, lead, b, cfg, width):
    """Run gcg_orth_recursive / gcg_orth_against; returns OrthOutcome (kept may be 0)."""
    o = _lib.OrthOpts(cfg.svd_leaf if cfg.svd_leaf is not None else 0, float(cfg.reorth_tol),
                      float(cfg.dependence_tol), int(cfg.max_reorth_passes), 0)
    kept, red, nrep = C.c_int64(), C.c_int64(), C.c_int64()
    cap = 4 * width + 64
    rep = (C.c_int64 * cap)()
    bargs = (b.nnz, D._p(b.rowptr), D._p(b.colidx), D._p(b.val)) if b is not None else \
        (0, None, None, None)
    _lib.call(name, ops.dev.h, x.shape[0], D._p(x), D._ld(x), *lead, *bargs, C.byref(o),
              C.byref(kept), C.byref(red), rep, cap, C.byref(nrep))
    return OrthOutcome(int(kept.value), [int(v) for v in rep[:min(nrep.value, cap)]],
                       int(red.value))


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
    if cfg.svd_leaf is not None and cfg.svd_leaf < 1:
        raise InvalidShape(f"svd_leaf must be >= 1, got {cfg.svd_leaf}")
    if _native_ok(ops, b) and x.shape[0] > 0:
        out = _native("gcg_orth_recursive", ops, x, (lo, hi), b, cfg, hi - lo)
        if out.num_kept <= 0:
            raise AllDependent("every column in the block is linearly dependent")
        return out
    st = _State(ops, x, b, cfg, lo, hi)
    st.leaf_width = cfg.svd_leaf if cfg.svd_leaf is not None else min(hi - lo, 16)
    if st.leaf_width < 1:
        raise InvalidShape(f"svd_leaf must be >= 1, got {st.leaf_width}")
    _recurse_svd(st, lo, hi)
    kept = st.active_end - lo
    if kept <= 0:
        raise AllDependent("every column in the block is linearly dependent")
    return OrthOutcome(kept, st.replaced, st.reductions)


def _seed_local_norms(st):
    """orth.py:114-119: without B the squared column norms join the first round."""
    if st.b is None:
        lo, hi = st.start, st.active_end
        dd = st.dev.empty(hi - lo)
        st.ops.col_dots(st.x[:, lo:hi], st.x[:, lo:hi], dd)
        st.d[lo:hi] = dd.cpu().numpy()
        st.note_scale(st.d[lo:hi])


def _mgs_block(st, start, stop):
    """Column-by-column orthonormalisation of x[:, start:stop] (orth.py:229-269).

    One fused reduction per column: the Gram of x[:, j:stop] against B x_j gives
    the squared norm (first entry) and the projections onto the rest of the
    block; the normalisation and the rank-1 removal are device kernels."""
    cfg, dev, ops = st.cfg, st.dev, st.ops
    j = start
    while j < min(stop, st.active_end):
        stop = min(stop, st.active_end)
        col = st.x[:, j:j + 1]
        bcol = st.bdot(col)
        w = stop - j
        g = dev.empty(w, 1)
        ops.gram(st.x[:, j:stop], bcol, g)
        st.reductions += 1
        if j == st.start and st.reductions == 1:
            _seed_local_norms(st)
        gh = g[:, 0].cpu().numpy()
        nrm2, fwd = float(gh[0]), gh[1:]
        st.note_scale([nrm2])
        if nrm2 <= cfg.dependence_tol * st.scale:
            if not st.pull_rear(j):
                return
            if j > st.start:
                _deflate_against(st, st.x[:, st.start:j], j, j + 1)
            continue
        known = st.d[j]
        if np.isfinite(known) and nrm2 <= _REPAIR_RATIO * max(known, st.scale):
            _deflate_against(st, st.x[:, st.start:j], j, j + 1)
            st.d[j] = np.nan
            continue
        inv = 1.0 / np.sqrt(nrm2)
        D.col_scale(dev, torch.full((1,), inv, dtype=torch.float64, device=dev.device), col)
        if fwd.size:
            cf = fwd * inv
            D.lincomb(dev, col, torch.from_numpy(cf[None, :].copy()).pin_memory().to(
                dev.device, non_blocking=True),
                      st.x[:, j + 1:stop], alpha=-1.0, beta=1.0)
            st.d[j + 1:stop] = np.maximum(st.d[j + 1:stop] - cf * cf, 0.0)
        st.d[j] = 1.0
        j += 1


def _block_deflate(st, start, stop):
    """Repeat-until removal of the finished block from every later column (orth.py:272-301).

    R' = (rest' B block)' is written transposed by the Gram kernel, so the
    update rest -= block R' is one LinComb; the repeat test uses the host-tracked
    norm estimates as in the reference."""
    cfg, dev, ops = st.cfg, st.dev, st.ops
    passes = 0
    while passes < cfg.max_reorth_passes:
        stop = min(stop, st.active_end)
        nrest = st.active_end - stop
        if nrest <= 0 or stop <= start:
            return
        blk = st.x[:, start:stop]
        rest = st.x[:, stop:st.active_end]
        bblock = st.bdot(blk)
        rt = dev.empty(stop - start, nrest)
        ops.gram(rest, bblock, rt, transpose_out=True)
        st.reductions += 1
        passes += 1
        D.lincomb(dev, blk, rt, rest, alpha=-1.0, beta=1.0)
        lost = dev.empty(nrest)
        D.col_dots(dev, rt, rt, lost)
        D.deflate_status(dev, rt, lost, _DGKS_RATIO, st.status)  # status[0] = max |R|
        rec = torch.cat([st.status[:1], lost]).cpu().numpy()
        if float(rec[0]) <= cfg.reorth_tol:
            return
        lost_h = rec[1:]
        known = st.d[stop:st.active_end]
        with np.errstate(invalid="ignore"):
            risky = lost_h > _DGKS_RATIO * np.maximum(known, 1e-300)
        st.d[stop:st.active_end] = np.maximum(known - lost_h, 0.0)
        if not bool(np.any(risky[np.isfinite(known)])):
            return


def modified_block_orth(ops, x, x0=None, b=None, cfg=None):
    """Alg. 2: B-orthonormalise device block ``x`` in place, optionally against a fixed
    B-orthonormal basis ``x0`` (orth.py:304-336).  Kept columns end in x[:, :num_kept]."""
    ops = _as_ops(ops)
    cfg = cfg if cfg is not None else OrthConfig()
    m = x.shape[1]
    if m == 0:
        return OrthOutcome(0, [], 0)
    if x0 is not None and x0.shape[1] == 0:
        x0 = None
    if x0 is not None and x0.shape[0] != x.shape[0]:
        raise InvalidShape(f"basis dim {x0.shape[0]} != block dim {x.shape[0]}")
    bw = cfg.block_width if cfg.block_width is not None else min(max(m // 4, 1), 200)
    if bw < 1:
        raise InvalidShape(f"block_width must be >= 1, got {bw}")
    st = _State(ops, x, b, cfg, 0, m)
    st.track = True
    if x0 is not None:
        _deflate_against(st, x0, 0, m)
    start = 0
    while start < st.active_end:
        stop = min(start + bw, st.active_end)
        _mgs_block(st, start, stop)
        stop = min(stop, st.active_end)
        if stop < st.active_end:
            _block_deflate(st, start, stop)
        start = stop
    if st.active_end <= 0:
        raise AllDependent("every column in the block is linearly dependent")
    return OrthOutcome(st.active_end, st.replaced, st.reductions)


def orth_against(ops, x, basis, b=None, cfg=None):
    """Deflate ``x`` against ``basis``, Alg. 3, then deflate + SVQB the kept block (orth.py:339-372)."""
    ops = _as_ops(ops)
    cfg = cfg if cfg is not None else OrthConfig()
    if x.shape[1] == 0:
        return OrthOutcome(0, [], 0)
    have_basis = basis is not None and basis.shape[1] > 0
    if have_basis:
        if basis.shape[0] != x.shape[0]:
            raise InvalidShape(f"basis dim {basis.shape[0]} != block dim {x.shape[0]}")
    if _native_ok(ops, b) and x.shape[0] > 0:
        K = basis.shape[1] if have_basis else 0
        out = _native("gcg_orth_against", ops, x,
                      (x.shape[1], D._p(basis) if K else None, D._ld(basis) if K else 0, K),
                      b, cfg, x.shape[1])
        if out.num_kept <= 0:
            raise AllDependent("every column in the block is linearly dependent")
        return out
    st = _State(ops, x, b, cfg, 0, x.shape[1])
    if have_basis:
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
