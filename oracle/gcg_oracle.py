"""CPU oracle for the GCG hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference package `gcgeig`
(/root/reference/pkg/src/gcgeig) for exactly the functions on the B200 hot
path.  It exists so that parity can be checked on machines where the
reference is not installed (the GPU box).  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may import it;
the product package `paper_2111_06552_b200` never does.

Pinning: tests/test_oracle_pin.py checks this restatement against golden
vectors produced by running the real reference (tests/golden/make_golden.py,
run in the build container where /root/reference exists) and, when the
reference has been built into oracle/_ref, against the live reference.

Every function cites the reference file:line it restates.  Paths below are
relative to /root/reference/pkg/src/gcgeig/.

Layout conventions follow the reference: multivectors are (n, k) float64
arrays in Fortran order; column ranges are 0-based half-open unless noted.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse


class OracleError(Exception):
    """Raised where the reference raises a GcgError subclass."""


class AllDependentError(OracleError):
    """Reference: errors.AllDependent (errors.py:24)."""


# ---------------------------------------------------------------------------
# L1 kernels: _kernels/_numpy_impl.py:12-47 and _cy.pyx:11-65


def csr_matvec(indptr, indices, data, x, out=None):
    """out = A @ x for a CSR matrix (_numpy_impl.py:12-20, _cy.pyx:11-23).

    Each output entry is a sequential sum over the row's nonzeros in storage
    order, which is what both reference backends compute.
    """
    n = len(indptr) - 1
    sp = scipy.sparse.csr_matrix((data, indices, indptr), shape=(n, x.shape[0]))
    res = sp @ np.asarray(x)
    if out is None:
        return np.asfortranarray(res)
    out[...] = res
    return out


def inner_product(x, y, out=None, chunk=8192, deterministic=False):
    """out[r, c] = sum_i x[i, r] * y[i, c] (_numpy_impl.py:23-33, _cy.pyx:26-50)."""
    if out is None:
        out = np.zeros((x.shape[1], y.shape[1]), order="F")
    n = x.shape[0]
    if (not deterministic) or chunk <= 0 or chunk >= n:
        out[...] = x.T @ y
        return out
    acc = np.zeros(out.shape)
    for s in range(0, n, chunk):
        e = min(s + chunk, n)
        acc += x[s:e].T @ y[s:e]
    out[...] = acc
    return out


def axpby(alpha, x, beta, y):
    """y <- alpha x + beta y; beta == 0 never reads y (_numpy_impl.py:36-47)."""
    if beta == 0.0:
        y[...] = 0.0 if alpha == 0.0 else x * alpha
        return y
    if beta != 1.0:
        y *= beta
    if alpha != 0.0:
        y += alpha * x
    return y


# ---------------------------------------------------------------------------
# L2 operators: operators.py:75-165


class Csr:
    """A symmetric CSR operator (operators.py:75-114)."""

    def __init__(self, m):
        sp = scipy.sparse.csr_matrix(m, dtype=np.float64)
        sp.sum_duplicates()
        self.sp = sp
        self.dim = sp.shape[0]

    def apply(self, x):
        return np.asfortranarray(self.sp @ np.asarray(x))


def shifted_apply(a, b, theta, x):
    """(A - theta B) x, or (A - theta I) x when b is None (operators.py:149-156)."""
    out = a.apply(x)
    if theta != 0.0:
        out -= theta * (x if b is None else b.apply(x))
    return out


# ---------------------------------------------------------------------------
# dense helpers: dense.py:63-133


def fix_signs(v):
    """Largest-|entry| of each column made positive, first index on ties (dense.py:63-71)."""
    if v.size == 0:
        return v
    lead = np.argmax(np.abs(v), axis=0)
    s = np.sign(v[lead, np.arange(v.shape[1])])
    s[s == 0.0] = 1.0
    v *= s
    return v


def eig_full(m):
    """All eigenpairs ascending, sign-fixed (dense.py:74-82)."""
    w, v = scipy.linalg.eigh(np.asarray(m, dtype=np.float64))
    return w, fix_signs(np.asfortranarray(v))


def eig_range(m, lo, hi):
    """Eigenpairs lo..hi (1-based inclusive), sign-fixed (dense.py:85-117, serial path)."""
    w, v = scipy.linalg.eigh(np.asarray(m, dtype=np.float64), subset_by_index=[lo - 1, hi - 1])
    return w, fix_signs(np.asfortranarray(v))


gram_eig = eig_full  # dense.py:120-133 is the same factorisation of a Gram matrix


# ---------------------------------------------------------------------------
# L3 block CG: cg.py:33-99


@dataclass
class CgResult:
    iterations: int
    converged: np.ndarray
    frozen: np.ndarray
    relative_residuals: np.ndarray


def _coldot(x, y):
    return np.einsum("ij,ij->j", x, y)


def block_cg(apply, rhs, x0, max_iters=30, rel_tol=0.01):
    """k independent CG recurrences sharing one operator call per sweep (cg.py:33-99).

    Columns stop at rel_tol * ||r0||; a direction with p'Ap <= 0 freezes the
    column at its current iterate.
    """
    rhs = np.asfortranarray(rhs, dtype=np.float64)
    n, k = rhs.shape
    if x0 is None:
        x = np.zeros((n, k), order="F")
        r = rhs.copy()
    else:
        x = np.array(x0, dtype=np.float64, order="F")
        r = rhs - apply(x)
    rn0 = np.sqrt(_coldot(r, r))
    target = rel_tol * rn0
    conv = rn0 <= target
    frozen = np.zeros(k, dtype=bool)
    rn = rn0.copy()
    z = r.copy()          # cg.py:63-65 (no preconditioner: z is a copy of r)
    p = z.copy()
    rz = _coldot(r, z)
    sweeps = 0
    for _ in range(max_iters):
        act = np.flatnonzero(~conv & ~frozen)
        if act.size == 0:
            break
        sweeps += 1
        pa = np.asfortranarray(p[:, act])
        qa = apply(pa)
        den = _coldot(pa, qa)
        neg = den <= 0.0
        if neg.any():
            frozen[act[neg]] = True
            keep = ~neg
            act, pa, qa, den = act[keep], pa[:, keep], qa[:, keep], den[keep]
            if act.size == 0:
                continue
        alpha = rz[act] / den
        x[:, act] += pa * alpha
        r[:, act] -= qa * alpha
        # distinct gathered copies, as in cg.py:86 (einsum rounds differently
        # when both operands are the same object)
        rn[act] = np.sqrt(_coldot(r[:, act], r[:, act]))
        fin = rn[act] <= target[act]
        conv[act[fin]] = True
        act = act[~fin]
        if act.size == 0:
            continue
        za = r[:, act]
        rz_new = _coldot(r[:, act], za)
        p[:, act] = za + p[:, act] * (rz_new / rz[act])
        rz[act] = rz_new
    return x, CgResult(sweeps, conv, frozen, rn / np.where(rn0 > 0.0, rn0, 1.0))


# ---------------------------------------------------------------------------
# L3 B-orthogonalisation: orth.py:124-226, 339-372


@dataclass
class OrthParams:
    """orth.OrthConfig defaults (orth.py:48-62)."""

    block_width: int | None = None
    svd_leaf: int | None = None
    reorth_tol: float = 1e-10
    dependence_tol: float = 1e-10
    max_reorth_passes: int = 3


DGKS = 0.5  # orth.py:43
REPAIR = 1e-8  # orth.py:45


class _State:
    """Per-call bookkeeping (orth.py:72-108)."""

    def __init__(self, x, b, prm, lo, hi):
        self.x, self.b, self.prm = x, b, prm
        self.lo0, self.end = lo, hi
        self.nred = 0
        self.replaced = []
        self.scale = 0.0
        self.d = np.full(x.shape[1], np.nan)
        self.leaf = 16

    def bmul(self, y):
        return y if self.b is None else self.b.apply(np.asfortranarray(y))

    def bump_scale(self, vals):
        self.scale = max(self.scale, float(np.max(vals, initial=0.0)))

    def rear_fill(self, slot):
        """orth.py:95-108: move the rearmost live column into `slot`."""
        self.replaced.append(slot)
        if self.end - 1 > slot:
            self.end -= 1
            self.x[:, slot] = self.x[:, self.end]
            self.d[slot] = self.d[self.end]
            return True
        self.end = slot
        return False


def deflate(st, basis, lo, hi):
    """Repeat-until projection of x[:, lo:hi] out of span(basis) (orth.py:124-152)."""
    prm = st.prm
    npass = 0
    while npass < prm.max_reorth_passes:
        hi = min(hi, st.end)
        if lo >= hi or basis.shape[1] == 0:
            return npass
        t = st.x[:, lo:hi]
        bt = st.bmul(t)
        coef = basis.T @ bt
        dn = np.einsum("ij,ij->j", t, bt)
        st.nred += 1
        npass += 1
        st.bump_scale(dn)
        t -= basis @ coef
        if float(np.abs(coef).max(initial=0.0)) <= prm.reorth_tol:
            st.d[lo:hi] = np.maximum(dn, 0.0)
            return npass
        lost = np.einsum("ij,ij->j", coef, coef)
        st.d[lo:hi] = np.maximum(dn - lost, 0.0)
        if not np.any(lost > DGKS * np.maximum(dn, 1e-300)):
            return npass
    return npass


def leaf_svqb(st, lo, hi):
    """Scaled-Gram orthonormalisation of a leaf block (orth.py:155-188)."""
    prm = st.prm
    npass = 0
    while True:
        hi = min(hi, st.end)
        if lo >= hi:
            return
        blk = st.x[:, lo:hi]
        g = blk.T @ st.bmul(blk)
        st.nred += 1
        npass += 1
        if np.abs(g - np.eye(hi - lo)).max() <= prm.reorth_tol:
            return
        w, v = gram_eig((g + g.T) / 2.0)
        st.bump_scale(w)
        floor = prm.dependence_tol * max(float(w.max(initial=0.0)), 0.0)
        nbad = int(np.searchsorted(w, floor, side="right"))
        if nbad == 0:
            blk[...] = blk @ (v / np.sqrt(w))
            if npass >= prm.max_reorth_passes:
                return
            continue
        keep = hi - lo - nbad
        if keep > 0:
            blk[:, :keep] = blk @ (v[:, nbad:] / np.sqrt(w[nbad:]))
        for slot in range(lo + keep, hi):
            if not st.rear_fill(slot):
                break
        npass = 0


def _recurse(st, lo, hi):
    """orth.py:191-204."""
    hi = min(hi, st.end)
    if lo >= hi:
        return
    width = hi - lo
    if width <= st.leaf:
        leaf_svqb(st, lo, hi)
        return
    mid = lo + width // 2
    _recurse(st, lo, mid)
    mid = min(mid, st.end)
    if lo < mid < st.end:
        deflate(st, st.x[:, lo:mid], mid, hi)
    _recurse(st, mid, hi)


@dataclass
class OrthResult:
    num_kept: int
    replaced_indices: list = field(default_factory=list)
    reduction_count: int = 0


def recursive_orth_svd(x, s=None, e=None, b=None, prm=None):
    """Alg. 3 on columns s..e (1-based inclusive) of x, in place (orth.py:207-226)."""
    prm = prm or OrthParams()
    s = 1 if s is None else s
    e = x.shape[1] if e is None else e
    if not (1 <= s <= e <= x.shape[1]):
        raise OracleError(f"bad range {s}..{e}")
    st = _State(x, b, prm, s - 1, e)
    st.leaf = prm.svd_leaf if prm.svd_leaf is not None else min(e - s + 1, 16)
    _recurse(st, s - 1, e)
    kept = st.end - (s - 1)
    if kept <= 0:
        raise AllDependentError("all columns dependent")
    return OrthResult(kept, st.replaced, st.nred)


def orth_against(x, basis, b=None, prm=None):
    """Deflate vs basis, Alg. 3, then deflate + SVQB the kept block again (orth.py:339-372)."""
    prm = prm or OrthParams()
    k = x.shape[1]
    if k == 0:
        return OrthResult(0, [], 0)
    st = _State(x, b, prm, 0, k)
    use_basis = basis is not None and basis.shape[1] > 0
    if use_basis:
        deflate(st, basis, 0, k)
    inner = recursive_orth_svd(x, 1, k, b=b, prm=prm)
    kept = inner.num_kept
    replaced = list(inner.replaced_indices)
    extra = 0
    if use_basis and kept > 0:
        post = _State(x, b, prm, 0, kept)
        deflate(post, basis, 0, kept)
        leaf_svqb(post, 0, kept)
        kept = post.end
        replaced += post.replaced
        extra = post.nred
        if kept <= 0:
            raise AllDependentError("all columns dependent")
    return OrthResult(kept, replaced, st.nred + inner.reduction_count + extra)


def _seed_norms(st):
    """orth.py:114-119: without B, every squared column norm joins the first round."""
    if st.b is None:
        sl = slice(st.lo0, st.end)
        st.d[sl] = np.einsum("ij,ij->j", st.x[:, sl], st.x[:, sl])
        st.bump_scale(st.d[sl])


def mgs_block(st, j0, j1):
    """Column-at-a-time orthonormalisation of x[:, j0:j1] (orth.py:229-269): one fused
    round per column (its squared B-norm + projections onto the rest of the block)."""
    prm = st.prm
    j = j0
    while j < min(j1, st.end):
        j1 = min(j1, st.end)
        c = st.x[:, j:j + 1]
        bc = st.bmul(c)
        nn = float(np.vdot(c, bc))
        proj = st.x[:, j + 1:j1].T @ bc
        st.nred += 1
        if j == st.lo0 and st.nred == 1:
            _seed_norms(st)
        st.bump_scale([nn])
        if nn <= prm.dependence_tol * st.scale:
            if not st.rear_fill(j):
                return
            if j > st.lo0:
                deflate(st, st.x[:, st.lo0:j], j, j + 1)
            continue
        tracked = st.d[j]
        if np.isfinite(tracked) and nn <= REPAIR * max(tracked, st.scale):
            deflate(st, st.x[:, st.lo0:j], j, j + 1)
            st.d[j] = np.nan
            continue
        s = 1.0 / np.sqrt(nn)
        c *= s
        if proj.size:
            st.x[:, j + 1:j1] -= c @ (proj.T * s)
            gone = (proj[:, 0] * s) ** 2
            st.d[j + 1:j1] = np.maximum(st.d[j + 1:j1] - gone, 0.0)
        st.d[j] = 1.0
        j += 1


def block_deflate(st, j0, j1):
    """Repeat-until sweep of the finished block x[:, j0:j1] out of all later columns
    (orth.py:272-301); tracked norm estimates drive the repeat test."""
    prm = st.prm
    npass = 0
    while npass < prm.max_reorth_passes:
        j1 = min(j1, st.end)
        later = st.x[:, j1:st.end]
        if later.shape[1] == 0 or j1 <= j0:
            return
        bb = st.bmul(st.x[:, j0:j1])
        r = later.T @ bb
        st.nred += 1
        npass += 1
        later -= st.x[:, j0:j1] @ r.T
        if float(np.abs(r).max(initial=0.0)) <= prm.reorth_tol:
            return
        gone = np.einsum("ij,ij->i", r, r)
        tracked = st.d[j1:st.end]
        with np.errstate(invalid="ignore"):
            risky = gone > DGKS * np.maximum(tracked, 1e-300)
        st.d[j1:st.end] = np.maximum(tracked - gone, 0.0)
        if not bool(np.any(risky[np.isfinite(tracked)])):
            return


def modified_block_orth(x, x0=None, b=None, prm=None):
    """Alg. 2 (orth.py:304-336): optional deflation against x0, then per block of width
    bw an MGS pass and a sweep of the block out of the remaining columns."""
    prm = prm or OrthParams()
    m = x.shape[1]
    if m == 0:
        return OrthResult(0, [], 0)
    if x0 is not None and x0.shape[1] == 0:
        x0 = None
    if x0 is not None and x0.shape[0] != x.shape[0]:
        raise OracleError("basis row count differs")
    bw = prm.block_width if prm.block_width is not None else min(max(m // 4, 1), 200)
    if bw < 1:
        raise OracleError(f"block width {bw}")
    st = _State(x, b, prm, 0, m)
    if x0 is not None:
        deflate(st, x0, 0, m)
    j0 = 0
    while j0 < st.end:
        j1 = min(j0 + bw, st.end)
        mgs_block(st, j0, j1)
        j1 = min(j1, st.end)
        if j1 < st.end:
            block_deflate(st, j0, j1)
        j0 = j1
    if st.end <= 0:
        raise AllDependentError("all columns dependent")
    return OrthResult(st.end, st.replaced, st.nred)


# ---------------------------------------------------------------------------
# L4 driver: solver.py:106-486


@dataclass
class OracleConfig:
    """solver.SolverConfig fields used on the hot path (solver.py:56-74).

    `init` and `residual` are the two parity switches of SURVEY §8(c):
    init="uniform" is the reference's mv_set_random (multivec.py:46-50),
    init="normal" the BASELINE N(0,1) block; residual="reference" is
    solver._rel_residual (solver.py:129-141), residual="relative" the
    north-star ||Ax - lam Bx|| / (|lam| ||Bx||).
    """

    num_eigen: int = 1
    tol: float = 1e-8
    block_size: int | None = None
    size_x: int | None = None
    max_gcg_iters: int = 1000
    cg_max_iters: int = 30
    cg_rel_tol: float = 0.01
    shift_mode: str = "dynamic"
    moving: bool = False
    seed: int = 0
    orth: OrthParams = field(default_factory=OrthParams)
    init: str = "uniform"
    residual: str = "reference"


@dataclass
class IterInfo:
    iteration: int
    num_converged: int
    first_unconverged_residual: float
    theta: float
    cg_iterations: int
    basis_size: int
    orth_reductions: int


@dataclass
class OracleReport:
    status: str
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray
    num_converged: int
    iterations: int
    residuals: np.ndarray
    history: list
    max_projection_dim: int
    total_reductions: int


def fill_random(x, seed, init="uniform"):
    """multivec.mv_set_random (multivec.py:46-50); init="normal" is the BASELINE draw."""
    g = np.random.Generator(np.random.PCG64(seed))
    if init == "normal":
        x[...] = g.standard_normal(x.shape)
    else:
        x[...] = g.uniform(-1.0, 1.0, size=x.shape)
    return x


def shift_for(mode, lam, nlocked, store_vals=()):
    """solver.select_shift (solver.py:113-126)."""
    if mode not in ("dynamic", "none"):
        raise OracleError(f"unknown shift mode {mode!r}")
    if mode == "none":
        return 0.0
    best = float(lam[nlocked - 1]) if nlocked > 0 else None
    for vals in store_vals:
        if len(vals):
            t = float(vals[-1])
            best = t if best is None or t > best else best
    return 0.0 if best is None else best


def rel_residual(ax, x, bx, lam, generalized, kind="reference"):
    """solver._rel_residual (solver.py:129-141) or the north-star criterion."""
    if kind == "relative":
        r = ax - lam * bx
        den = abs(lam) * math.sqrt(float(bx @ bx))
    elif generalized:
        r = ax - lam * bx
        den = math.sqrt(max(float(x @ bx), 0.0))
        if lam > 0.0:
            den *= lam
    else:
        r = ax - lam * x
        den = math.sqrt(float(x @ x))
    if den == 0.0:
        den = 1.0
    return math.sqrt(float(r @ r)) / den


def converged_prefix(a, b, xn, lam, limit, chunk, tol, kind):
    """solver._count_converged (solver.py:144-164)."""
    cnt = 0
    for s in range(0, limit, chunk):
        e = min(s + chunk, limit)
        xc = np.asfortranarray(xn[:, s:e])
        axc = a.apply(xc)
        bxc = b.apply(xc) if b is not None else xc
        for j in range(e - s):
            rr = rel_residual(axc[:, j], xc[:, j], bxc[:, j], float(lam[s + j]), b is not None, kind)
            if rr < tol:
                cnt += 1
            else:
                return cnt, rr
    return cnt, 0.0


def momentum_coeffs(coeffs, nx, g0, gw, dep_tol):
    """solver._build_p (solver.py:167-199)."""
    m = coeffs.shape[0]
    if gw <= 0 or m <= nx:
        return None
    pt = coeffs[:, g0:g0 + gw].copy()
    pt[:nx, :] = 0.0
    for _ in range(2):
        pt -= coeffs @ (coeffs.T @ pt)
    g = pt.T @ pt
    w, v = gram_eig((g + g.T) / 2.0)
    nbad = int(np.searchsorted(w, dep_tol * max(float(w.max(initial=0.0)), 0.0), side="right"))
    if nbad >= gw:
        return None
    q = pt @ (v[:, nbad:] / np.sqrt(w[nbad:]))
    q -= coeffs @ (coeffs.T @ q)
    g = q.T @ q
    w, v = gram_eig((g + g.T) / 2.0)
    nbad = int(np.searchsorted(w, 1e-4 * max(float(w.max(initial=0.0)), 0.0), side="right"))
    if nbad >= q.shape[1]:
        return None
    return q @ (v[:, nbad:] / np.sqrt(w[nbad:]))


def gcg_solve(a, b=None, cfg=None):
    """solver.gcg_solve (solver.py:226-486), control flow restated line for line.

    `a`, `b` are scipy sparse matrices (or None for b).
    """
    cfg = cfg or OracleConfig()
    A = Csr(a)
    B = Csr(b) if b is not None else None
    n = A.dim
    ne = int(cfg.num_eigen)
    if not 1 <= ne <= n:
        raise OracleError("num_eigen out of range")
    bs = cfg.block_size if cfg.block_size is not None else max(1, math.ceil(ne / 5))
    bs = min(bs, n)
    if cfg.moving:
        sx = min(3 * bs, n)
    else:
        sx = cfg.size_x if cfg.size_x is not None else min(ne + 3 * bs, n)
        sx = min(max(sx, ne), n)
    prm = cfg.orth
    rnd = lambda blk, seed: fill_random(blk, seed, cfg.init)  # noqa: E731

    v = np.zeros((n, sx + 2 * bs), order="F")
    lam = np.zeros(sx + 2 * bs)
    rnd(v[:, :sx], cfg.seed)
    o = recursive_orth_svd(v, 1, sx, b=B, prm=prm)
    total_red = o.reduction_count
    if o.num_kept < sx:
        rnd(v[:, o.num_kept:sx], cfg.seed + 9973)
        o = recursive_orth_svd(v, 1, sx, b=B, prm=prm)
        total_red += o.reduction_count
        if o.num_kept < sx:
            raise AllDependentError("could not build a full-rank starting block")

    locked, npc, nwc = 0, 0, 0
    abar_prev, p_coupling = None, None
    store_x, store_vals = [], []
    history = []
    max_m = 0
    status = "max_iterations"
    its = 0
    for it in range(1, cfg.max_gcg_iters + 1):
        its = it
        d = sx - locked
        m = d + npc + nwc
        max_m = max(max_m, m)
        basis = v[:, locked:sx + npc + nwc]
        # STEP 3: projected matrix (solver.py:277-290)
        if abar_prev is None:
            abar = basis.T @ A.apply(basis)
        else:
            abar = np.zeros((m, m), order="F")
            abar[:d, :d] = np.diag(lam[locked:sx])
            if npc:
                abar[d:d + npc, d:d + npc] = p_coupling
            if nwc:
                aw = A.apply(v[:, sx + npc:sx + npc + nwc])
                cross = basis.T @ aw
                abar[:, d + npc:] = cross
                abar[d + npc:, :] = cross.T
        abar = (abar + abar.T) / 2.0
        lam_new, coeffs = eig_range(abar, 1, d)
        x_new = np.asfortranarray(basis @ coeffs)
        # STEP 4: converged prefix (solver.py:302-323)
        stored = sum(len(s) for s in store_vals)
        limit = max(0, min(sx - locked, ne - stored - locked))
        newly, first_res = converged_prefix(A, B, x_new, lam_new, limit, bs, cfg.tol, cfg.residual)
        c = locked + newly
        total_locked = stored + c
        if total_locked >= ne:
            v[:, locked:sx] = x_new
            lam[locked:sx] = lam_new
            locked = c
            status = "converged"
            history.append(IterInfo(it, total_locked, first_res,
                                    shift_for(cfg.shift_mode, lam, locked, store_vals), 0, m, 0))
            break
        compacted = refilled = False
        iter_red = 0
        # moving window (solver.py:325-363)
        if cfg.moving and c > 0 and (c >= 2 * bs or c >= sx):
            wf, vf = eig_full(abar)
            x_all = np.asfortranarray(basis @ vf)
            store_x.append(np.asfortranarray(np.hstack([v[:, :locked], x_all[:, :newly]])))
            store_vals.append(np.concatenate([lam[:locked], wf[:newly]]))
            stored += c
            sx = m - newly
            if sx:
                v[:, :sx] = x_all[:, newly:]
                lam[:sx] = wf[newly:]
            locked, npc, nwc = 0, 0, 0
            p_coupling = None
            compacted = True
            c = 0
            if sx < bs:
                add = min(3 * bs, n - stored) - sx
                if add > 0:
                    rnd(v[:, sx:sx + add], cfg.seed + 104729 * it)
                    defl = np.asfortranarray(np.hstack(store_x + [v[:, :sx]]))
                    ro = orth_against(v[:, sx:sx + add], defl, b=B, prm=prm)
                    iter_red += ro.reduction_count
                    sx += ro.num_kept
                refilled = True
                if sx <= 0:
                    raise AllDependentError("moving window could not be refilled")
        theta = shift_for(cfg.shift_mode, lam, locked, store_vals)
        cg_its = 0
        if not refilled:
            # STEP 5 (solver.py:367-384)
            if compacted:
                bs_eff = max(1, min(bs, ne - stored, sx))
            else:
                bs_eff = max(1, min(bs, ne - stored - c, sx - c))
                phat = momentum_coeffs(coeffs, d, c - locked, bs_eff, prm.dependence_tol)
                if phat is None:
                    p_new, p_coupling = None, None
                else:
                    p_new = np.asfortranarray(basis @ phat)
                    p_coupling = phat.T @ (abar @ phat)
                v[:, locked:sx] = x_new
                lam[locked:sx] = lam_new
                locked = c
                npc = 0 if p_new is None else p_new.shape[1]
                if npc:
                    v[:, sx:sx + npc] = p_new
            # STEP 6: damped inverse power (solver.py:386-396)
            xa = np.asfortranarray(v[:, locked:locked + bs_eff])
            la = lam[locked:locked + bs_eff]
            bxa = B.apply(xa) if B is not None else xa.copy()
            rhs = np.asfortranarray(bxa * (la - theta))
            if theta == 0.0:
                op = A.apply
            else:
                op = lambda y, _t=theta: shifted_apply(A, B, _t, y)  # noqa: E731
            w_raw, cg = block_cg(op, rhs, xa, cfg.cg_max_iters, cfg.cg_rel_tol)
            cg_its = cg.iterations
            # STEP 2: W against [store, X, P] (solver.py:398-420)
            wreg = v[:, sx + npc:sx + npc + bs_eff]
            wreg[...] = w_raw
            if store_x:
                defl = np.asfortranarray(np.hstack(store_x + [v[:, :sx + npc]]))
            else:
                defl = v[:, :sx + npc]
            try:
                wo = orth_against(wreg, defl, b=B, prm=prm)
                nwc = wo.num_kept
                iter_red += wo.reduction_count
            except AllDependentError:
                nwc = 0
            if nwc == 0:
                rnd(wreg, cfg.seed + 7919 * it)
                try:
                    wo = orth_against(wreg, defl, b=B, prm=prm)
                    nwc = wo.num_kept
                    iter_red += wo.reduction_count
                except AllDependentError:
                    nwc = 0
        total_red += iter_red
        abar_prev = None if refilled else abar
        history.append(IterInfo(it, total_locked, first_res, theta, cg_its, m, iter_red))

    # result assembly (solver.py:447-472)
    if store_x:
        ax_all = np.asfortranarray(np.hstack(store_x + [v[:, :locked]]))
        av = np.concatenate(store_vals + [lam[:locked]])
        n_conv = av.shape[0]
        if n_conv < ne:
            extra = min(ne - n_conv, sx - locked)
            ax_all = np.asfortranarray(np.hstack([ax_all, v[:, locked:locked + extra]]))
            av = np.concatenate([av, lam[locked:locked + extra]])
        take = min(ne, av.shape[0])
        vals = av[:take].copy()
        vecs = np.asfortranarray(ax_all[:, :take])
    else:
        n_conv = locked
        vals = lam[:ne].copy()
        vecs = np.asfortranarray(v[:, :ne])
    res = np.empty(vals.shape[0])
    if vals.shape[0]:
        axv = A.apply(vecs)
        bxv = B.apply(vecs) if B is not None else vecs
        for j in range(vals.shape[0]):
            res[j] = rel_residual(axv[:, j], vecs[:, j], bxv[:, j], float(vals[j]), B is not None,
                                  cfg.residual)
    return OracleReport(status, vals, vecs, min(n_conv, ne), its, res, history, max_m, total_red)
