"""GCG eigensolver driver with every long-vector operation on the B200.

Drop-in for the reference entry point ``gcg_solve(a, b=None, config=None) ->
SolverReport`` (solver.py:226-486): same SolverConfig fields and defaults,
same control flow (Alg. 1 STEPs 2-6, locking, dynamic shift, moving window),
same report.  The multivector arena V = [X | P | W] (n x (sx + 2 bs)) lives in
HBM, row-major; the host only ever sees m x m-sized decisions (eigenvalues,
residual norms, dependence counts) read back as a handful of doubles.

The same driver runs row-partitioned over several GPUs (``gcg_solve_distributed``):
the multivector operations go through an ops object (mvops.LocalOps on one GPU,
distributed.DistOps across ranks) that adds halo exchanges and ordered
reductions; every host-side decision is taken on bit-identical replicated data.

Two parity switches that the reference does not have:
``init`` ("uniform" = reference mv_set_random, "normal" = BASELINE N(0,1)) and
``residual`` ("reference" = solver._rel_residual, "relative" = north-star
||Ax - lam Bx|| / (|lam| ||Bx||)).
"""

from __future__ import annotations

import os

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import device as D
from .dense import sym_eig_full, sym_eig_range_split
from .mvops import PrefaultedHost

# GCG_PY_BUILD_P=1: the Python driver for the momentum block (A/B and debugging)
_PY_BUILD_P = os.environ.get("GCG_PY_BUILD_P", "0") == "1"
from .errors import AllDependent, InvalidShape
from .mvops import LocalOps
from .operators import DeviceProblem, as_device_problem
from .orth import OrthConfig, orth_against, recursive_orth_svd

__all__ = [
    "SolverConfig",
    "IterationRecord",
    "SolverReport",
    "gcg_solve",
    "gcg_solve_ops",
    "select_shift",
    "moving_memory_budget",
    "device_memory_plan",
]

BACKEND_NAME = "sm100"
_TIMING_KEYS = ("t_step2", "t_step3", "t_step4", "t_step5", "t_step6")
_RESIDUAL_MODES = {"reference": None, "relative": 2}
_RNG_CHUNK_ROWS = 1 << 16
_PANEL_BYTES = 512 << 20      # row-panel scratch of the wide in-place LinComb
_PANEL_MIN_ROWS = 1 << 16
_AB_CHUNK_BYTES = 4 << 30     # A*basis of the full projection in column chunks above this


@dataclass
class SolverConfig:
    """solver.SolverConfig (solver.py:56-74) + the two parity switches."""

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
    deterministic: bool = False
    orth: OrthConfig = field(default_factory=OrthConfig)
    collect_history: bool = True
    stall_window: int = 50
    instrument_orth: bool = False
    cross_check_abar: bool = False
    # B200 drop-in extensions
    init: str = "uniform"          # "uniform" (reference) | "normal" (BASELINE, host PCG64)
    #                                | "philox" (seeded N(0,1) drawn on the device per global row)
    residual: str = "reference"    # "reference" | "relative" (north-star)
    validate: bool = True          # host symmetry/finiteness check of the input matrices
    return_device: bool = False    # keep eigenvectors as a device tensor (row-major n x nev)
    rr_split: bool = False         # distributed: split the RR index range over ranks (§8(f) 4)


@dataclass
class IterationRecord:
    iteration: int
    num_converged: int
    first_unconverged_residual: float
    theta: float
    cg_iterations: int
    basis_size: int
    orth_reductions: int
    timings: dict = field(default_factory=dict)
    basis_defect: float | None = None
    abar_defect: float | None = None


@dataclass
class SolverReport:
    status: str
    eigenvalues: np.ndarray
    eigenvectors: object
    num_converged: int
    iterations: int
    residuals: np.ndarray
    history: list
    stagnated: bool
    max_projection_dim: int
    total_reductions: int
    backend: str
    row_range: tuple = (0, 0)      # rows of `eigenvectors` (all of them on one GPU)


def moving_memory_budget(size_x, block_size):
    """solver.moving_memory_budget (solver.py:106-110)."""
    mpd = size_x + 2 * block_size
    return (size_x + 2 * block_size) + 2 * mpd * mpd + 10 * mpd + size_x * block_size


def device_memory_plan(n_local, nnz_local, num_eigen, block_size=None, size_x=None,
                       moving=False, nghost=0, generalized=False):
    """Peak HBM bytes of one rank's solve (this implementation's allocations).

    The arena [store | X | P | W] (moving: nev + sx + 2bs columns, else sx + 2bs) and the
    block-CG workspace (r and x with ghost rows, p and q) are live for the whole solve;
    on top of them at most three n_local x max(bs, 256) temporaries (residual chunk,
    its A*x, the CG right-hand side / Ritz chunk) and the 512 MB panel scratch of the
    wide in-place LinComb.  Returns a dict of the terms and their sum."""
    bs = block_size if block_size is not None else max(1, math.ceil(num_eigen / 5))
    if moving:
        sx = 3 * bs
    else:
        sx = size_x if size_x is not None else num_eigen + 3 * bs
    rows = n_local + nghost
    arena = 8 * rows * ((num_eigen if moving else 0) + sx + 2 * bs)
    csr = 4 * (n_local + 1) + 12 * nnz_local + (8 * nnz_local if generalized else 0)
    cg = 8 * bs * (2 * rows + 2 * n_local)
    temps = 3 * 8 * n_local * max(bs, 256)
    if generalized:
        temps += 8 * n_local * bs  # B * block in the orthogonalisation
    plan = {"csr": csr, "arena": arena, "cg": cg, "temporaries": temps,
            "panel": _PANEL_BYTES}
    plan["total"] = sum(plan.values())
    return plan


def select_shift(mode, lam, num_locked, store_vals=()):
    """solver.select_shift (solver.py:113-126): largest locked eigenvalue, else 0."""
    if mode not in ("dynamic", "none"):
        raise InvalidShape(f"unknown shift mode {mode!r}")
    if mode == "none":
        return 0.0
    best = None
    if num_locked > 0:
        best = float(lam[num_locked - 1])
    for vals in store_vals:
        if len(vals):
            top = float(vals[-1])
            best = top if best is None or top > best else best
    return 0.0 if best is None else best


def _stagnation_flag(history, window):
    """solver._stagnation_flag (solver.py:202-210)."""
    if window <= 0 or len(history) < window:
        return False
    tail = history[-window:]
    if tail[-1].num_converged != tail[0].num_converged:
        return False
    return not (tail[-1].first_unconverged_residual < 0.9 * tail[0].first_unconverged_residual)


def _h2d(dev, arr):
    """Small host vector -> device without a host sync: staged through pinned memory
    (torch's caching host allocator) and copied asynchronously on the solver stream.
    A pageable-memory copy would wait for all queued device work first."""
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).pin_memory().to(
        dev.device, non_blocking=True)


class _LazyMarks(dict):
    """The per-step times of one iteration record: a dict whose CUDA-event intervals
    are resolved on first read (after the solve), so returning the report does not
    wait on ~300 event-timing calls inside the caller's timed region."""

    def _resolve(self):
        t = self.__dict__.pop("_timer", None)
        if t is not None:
            t.resolve()

    def __getitem__(self, k):
        self._resolve()
        return dict.__getitem__(self, k)

    def get(self, k, default=None):
        self._resolve()
        return dict.get(self, k, default)

    def __iter__(self):
        self._resolve()
        return dict.__iter__(self)

    def items(self):
        self._resolve()
        return dict.items(self)

    def keys(self):
        self._resolve()
        return dict.keys(self)

    def values(self):
        self._resolve()
        return dict.values(self)

    def copy(self):
        self._resolve()
        return dict(self)

    def __repr__(self):
        self._resolve()
        return dict.__repr__(self)

    def __eq__(self, other):
        self._resolve()
        return dict.__eq__(self, other)

    __hash__ = None


class _Timer:
    """Per-step GPU time of one iteration (the reference's t_step* wall clocks,
    solver.py:269-445): a CUDA event is recorded on the solver stream at every step
    boundary and the intervals are resolved once after the loop, so the timings
    measure device work and add no host synchronisation inside the iteration.
    Disabled (all zero) in deterministic mode, as in the reference."""

    def __init__(self, enabled, stream):
        self.enabled = enabled and stream is not None
        self.marks = _LazyMarks({k: 0.0 for k in _TIMING_KEYS})
        if self.enabled:
            self.marks._timer = self
        self._stream = stream
        self._laps = []
        self._last = self._event() if self.enabled else None

    def _event(self):
        e = torch.cuda.Event(enable_timing=True)
        e.record(self._stream)
        return e

    def lap(self, key):
        if self.enabled:
            now = self._event()
            self._laps.append((key, self._last, now))
            self._last = now

    def resolve(self):
        self.marks.__dict__.pop("_timer", None)
        for key, e0, e1 in self._laps:
            e1.synchronize()
            dict.__setitem__(self.marks, key, dict.__getitem__(self.marks, key) +
                             e0.elapsed_time(e1) / 1e3)
        self._laps = []


class _Solve:
    """State of one device solve (the body of solver.py:226-486)."""

    def __init__(self, ops, cfg):
        self.ops = ops
        self.dev = ops.dev
        self.prob = ops.prob
        self.cfg = cfg
        self.generalized = self.prob.B is not None
        if cfg.init not in ("uniform", "normal", "philox"):
            raise InvalidShape(f"unknown init {cfg.init!r}")
        mode = _RESIDUAL_MODES.get(cfg.residual, "bad")
        if mode == "bad":
            raise InvalidShape(f"unknown residual kind {cfg.residual!r}")
        self.res_mode = mode if mode is not None else (1 if self.generalized else 0)
        self.scalar = self.dev.empty(8)

    # -- small helpers -------------------------------------------------------
    def set_random(self, block, seed):
        """multivec.mv_set_random (multivec.py:46-50) on host, uploaded (parity).

        The global n x k block is drawn in row order (row chunks consume the
        PCG64 stream exactly like one call); each rank keeps its own rows.
        """
        ops = self.ops
        if self.cfg.init == "philox":  # device draw: same global block for any row partition
            D.fill_normal(self.dev, block, ops.row0, seed)
            return
        rng = np.random.Generator(np.random.PCG64(seed))
        k = block.shape[1]
        r0, r1 = ops.row0, ops.row0 + ops.nloc
        for c0 in range(0, min(r1, ops.n_global), _RNG_CHUNK_ROWS):
            c1 = min(c0 + _RNG_CHUNK_ROWS, ops.n_global)
            shape = (c1 - c0, k)
            host = rng.standard_normal(shape) if self.cfg.init == "normal" else \
                rng.uniform(-1.0, 1.0, size=shape)
            lo, hi = max(c0, r0), min(c1, r1)
            if lo < hi:
                src = torch.from_numpy(host[lo - c0:hi - c0]).to(self.dev.device)
                D.copy(self.dev, src, block[lo - r0:hi - r0])

    def apply_a(self, x):
        return self.ops.apply(self.prob.A, x)

    def apply_b(self, x):
        return x if self.prob.B is None else self.ops.apply(self.prob.B, x)

    def residuals(self, x, lam_dev):
        """Per-column relative residuals of Ritz pairs (solver.py:129-141), device -> host."""
        k = x.shape[1]
        out = np.empty(k)
        for s in range(0, k, 256):
            e = min(s + 256, k)
            xc = x[:, s:e]
            ax = self.apply_a(xc)
            bx = self.apply_b(xc)
            r = self.dev.empty(e - s)
            self.ops.residuals(ax, xc, bx, lam_dev[s:e], self.res_mode, r)
            out[s:e] = self.ops.broadcast(r).cpu().numpy()
        return out

    def count_converged(self, basis, coeffs, lam_new_dev, limit, chunk, tol):
        """solver._count_converged (solver.py:144-164): prefix of Ritz pairs below tol.

        The Ritz vectors are formed chunk by chunk (basis @ coeffs[:, chunk]) only
        as far as the prefix test reads them; the full X update happens in place
        afterwards (:meth:`update_in_place`).
        The host copy of the Ritz values rides along with the first chunk's
        residuals (one device->host read instead of two); returns
        (count, first unconverged residual, Ritz values on the host)."""
        count = 0
        xc = None
        lam_host = None
        for start in range(0, limit, chunk):
            stop = min(start + chunk, limit)
            if xc is None or xc.shape[1] != stop - start:
                xc = self.ops.vec(stop - start)
            D.lincomb(self.dev, basis, coeffs[:, start:stop], xc)
            if lam_host is None and stop - start <= 256:
                r = self.residuals_dev(xc, lam_new_dev[start:stop])
                both = torch.cat([lam_new_dev, r]).cpu().numpy()
                lam_host, rel = both[:lam_new_dev.shape[0]], both[lam_new_dev.shape[0]:]
            else:
                rel = self.residuals(xc, lam_new_dev[start:stop])
            for j in range(stop - start):
                if rel[j] < tol:
                    count += 1
                else:
                    return count, float(rel[j]), lam_host
        return count, 0.0, lam_host

    def residuals_dev(self, x, lam_dev):
        """Relative residuals of up to 256 Ritz pairs as a replicated device vector."""
        ax = self.apply_a(x)
        bx = self.apply_b(x)
        r = self.dev.empty(x.shape[1])
        self.ops.residuals(ax, x, bx, lam_dev, self.res_mode, r)
        return self.ops.broadcast(r)

    def build_p(self, coeffs, num_x_rows, group_start, group_width, dep_tol):
        """solver._build_p (solver.py:167-199) on device; returns phat (m x np) or None."""
        dev = self.dev
        m = coeffs.shape[0]
        if group_width <= 0 or m <= num_x_rows:
            return None
        d = coeffs.shape[1]
        if self.ops.size == 1 and not _PY_BUILD_P:
            # native: same operations and decisions, two pinned host reads (gcg_build_p)
            return D.build_p(dev, coeffs, num_x_rows, group_start, group_width, dep_tol)
        pt = dev.empty(m, group_width)
        D.copy(dev, coeffs[:, group_start:group_start + group_width], pt)
        D.fill(dev, pt[:num_x_rows], 0.0)
        tmp = dev.empty(d, group_width)
        for _ in range(2):
            D.dgemm(dev, coeffs, pt, tmp, ta=True)
            D.dgemm(dev, coeffs, tmp, pt, alpha=-1.0, beta=1.0)
        q, kept = self._orthonormalize_small(pt, dep_tol)
        if q is None:
            return None
        tmp = dev.empty(d, kept)
        D.dgemm(dev, coeffs, q, tmp, ta=True)
        D.dgemm(dev, coeffs, tmp, q, alpha=-1.0, beta=1.0)
        q2, _ = self._orthonormalize_small(q, 1e-4)
        return q2

    def _orthonormalize_small(self, pt, rel):
        """g = pt'pt; symmetric eig; drop eigenvalues <= rel*max; pt V/sqrt(w)."""
        dev = self.dev
        gw = pt.shape[1]
        g = dev.empty(gw, gw)
        D.dgemm(dev, pt, pt, g, ta=True)
        D.symmetrize(dev, g)
        dec = sym_eig_full(dev, g)
        self.ops.broadcast(dec.values)
        self.ops.broadcast(dec.vectors)
        D.count_le(dev, dec.values, rel, self.scalar)
        bad = int(self.scalar[0].item())
        if bad >= gw:
            return None, 0
        kept = gw - bad
        scaled = dev.empty(gw, kept)
        D.scale_rsqrt(dev, dec.vectors, dec.values, bad, scaled)
        q = dev.empty(pt.shape[0], kept)
        D.dgemm(dev, pt, scaled, q)
        return q, kept

    def update_in_place(self, basis, cm, dst):
        """dst <- basis @ cm where dst = the leading columns of basis (the reference's
        v[:, locked:sx] = x_new; v[:, sx:sx+np] = p_new, solver.py:378-384, and the
        moving window's x_all = basis @ full.vectors, :333).  One in-place lincomb when
        all columns fit one CTA tile (<= 256); wider products go through row panels: each
        output row depends only on the same input row, so a panel scratch of
        _PANEL_BYTES replaces the n x d temporary (cfg5: 33.5 GB per rank at 4 GPUs)."""
        d = cm.shape[1]
        if d <= 256:
            D.lincomb(self.dev, basis, cm, dst)
            return
        nloc = basis.shape[0]
        rows = int(min(nloc, max(_PANEL_MIN_ROWS, _PANEL_BYTES // (8 * d))))
        tmp = self.dev.empty(rows, d)
        for r in range(0, nloc, rows):
            e = min(r + rows, nloc)
            D.lincomb(self.dev, basis[r:e], cm, tmp[:e - r])
            D.copy(self.dev, tmp[:e - r], dst[r:e])

    def projected(self, basis, abar):
        """abar = basis' A basis (solver.py:279); A basis in column chunks when the n x m
        product would be large (one chunk below _AB_CHUNK_BYTES: the round-1 path)."""
        m = basis.shape[1]
        step = m if basis.shape[0] * m * 8 <= _AB_CHUNK_BYTES else 256
        for c0 in range(0, m, step):
            c1 = min(m, c0 + step)
            ab = self.apply_a(basis[:, c0:c1])
            self.ops.gram(basis, ab, abar if step == m else abar[:, c0:c1])
            del ab
        D.symmetrize(self.dev, abar)


def gcg_solve(a, b=None, config=None, *, x0=None):
    """Run the block eigensolver on the B200; returns a :class:`SolverReport`.

    ``a``/``b``: scipy sparse or dense host matrices, or a prepared DeviceProblem
    (matrices already in HBM).  ``x0`` (optional, n x size_x, host array or device
    tensor) replaces the seeded initial draw — for callers that generate the
    seeded block once and reuse it (bench.py); the seeded refills are unchanged.
    """
    cfg = config if config is not None else SolverConfig()
    dev = D.default_context()
    if isinstance(a, DeviceProblem):
        prob = a
    else:
        prob = as_device_problem(dev, a, b, validate=cfg.validate)
    return gcg_solve_ops(LocalOps(dev, prob), cfg, x0=x0)


def gcg_solve_ops(ops, cfg, x0=None):
    """The GCG iteration (solver.py:226-486) over an ops object (one GPU or one rank)."""
    S = _Solve(ops, cfg)
    dev, prob = ops.dev, ops.prob
    n = ops.n_global
    nloc = ops.nloc
    ne = int(cfg.num_eigen)
    if not (1 <= ne <= n):
        raise InvalidShape(f"num_eigen must be in 1..{n}, got {ne}")
    if cfg.shift_mode not in ("dynamic", "none"):
        raise InvalidShape(f"unknown shift mode {cfg.shift_mode!r}")
    bs = cfg.block_size if cfg.block_size is not None else max(1, math.ceil(ne / 5))
    bs = min(bs, n)
    if cfg.moving:
        sx = min(3 * bs, n)
    else:
        sx = cfg.size_x if cfg.size_x is not None else min(ne + 3 * bs, n)
        sx = min(max(sx, ne), n)
    ocfg = cfg.orth
    det = cfg.deterministic
    Bop = prob.B

    # One arena for the converged store and the window (SURVEY §7 "Memory"):
    # columns [0, S) hold the pairs the moving window has emitted, the window
    # [X | P | W] starts at S.  [store, X, P] — the deflation basis of STEP 2 — is
    # then a contiguous column range, the window slide is an in-place LinComb plus
    # S += c, and nothing is copied (the reference hstacks, solver.py:337,356,401,450).
    width = (ne if cfg.moving else 0) + sx + 2 * bs
    arena = ops.vec(width, zero=True)
    S_off = 0
    v = arena
    lam = np.zeros(sx + 2 * bs)
    # host eigenvector buffer, page-faulted in the background during the solve
    host_out = None if cfg.return_device else PrefaultedHost(nloc, ne)
    if x0 is None:
        S.set_random(v[:, :sx], cfg.seed)
    else:
        if tuple(x0.shape) != (nloc, sx):
            raise InvalidShape(f"x0 shape {tuple(x0.shape)} != ({nloc}, {sx})")
        src = x0 if isinstance(x0, torch.Tensor) else torch.from_numpy(np.asarray(x0))
        if src.device != dev.device:
            src = src.to(dev.device, non_blocking=True)
        D.copy(dev, src.contiguous(), v[:, :sx])
    out = recursive_orth_svd(ops, v, 1, sx, b=Bop, cfg=ocfg)
    total_red = out.reduction_count
    if out.num_kept < sx:
        S.set_random(v[:, out.num_kept:sx], cfg.seed + 9973)
        out = recursive_orth_svd(ops, v, 1, sx, b=Bop, cfg=ocfg)
        total_red += out.reduction_count
        if out.num_kept < sx:
            raise AllDependent("could not build a full-rank starting block")

    locked = 0
    np_, nw = 0, 0
    abar_prev = None
    p_coupling = None
    store_vals = []
    history = []
    pending_cg = []
    timers = []
    max_m = 0
    status = "max_iterations"
    iters_run = 0
    # the next iteration's A W and [X P W]' A W, enqueued as soon as STEP 2 has fixed W
    # (before this iteration's bookkeeping), with the timer they are charged to
    pre_timer = pre_cross = None

    for it in range(1, cfg.max_gcg_iters + 1):
        iters_run = it
        timer = pre_timer if pre_timer is not None else \
            _Timer(not det and cfg.collect_history, getattr(dev, "stream", None))
        timers.append(timer)
        d = sx - locked
        m = d + np_ + nw
        max_m = max(max_m, m)
        basis = v[:, locked:sx + np_ + nw]

        # STEP 3: projected matrix (solver.py:277-294)
        abar = dev.empty(m, m)
        if abar_prev is None:
            S.projected(basis, abar)
        else:
            cross = pre_cross
            if nw and cross is None:
                aw = S.apply_a(v[:, sx + np_:sx + np_ + nw])
                cross = dev.empty(m, nw)
                ops.gram(basis, aw, cross)
            lam_x = _h2d(dev, lam[locked:sx])
            D.abar_assemble(dev, d, lam_x, p_coupling if np_ else None, cross, abar)
        pre_timer = pre_cross = None
        abar_defect = None
        if cfg.cross_check_abar and abar_prev is not None:
            naive = dev.empty(m, m)
            ops.gram(basis, S.apply_a(basis), naive)
            D.symmetrize(dev, naive)
            D.max_abs_diff(dev, abar, naive, S.scalar)
            abar_defect = float(S.scalar[0].item())

        if cfg.rr_split and ops.size > 1:
            # split-range RR: rank r solves a slice of 1..d, all-gather
            dec = sym_eig_range_split(ops, abar, 1, d)
            full = None
            lam_new_dev, coeffs = dec.values, dec.vectors
        else:
            full = sym_eig_full(dev, abar)
            ops.broadcast(full.values)      # every replica continues from rank 0's RR solution
            ops.broadcast(full.vectors)
            lam_new_dev = full.values[:d]
            coeffs = full.vectors[:, :d]
        timer.lap("t_step3")

        stored = sum(len(vv) for vv in store_vals)
        limit = max(0, min(sx - locked, ne - stored - locked))
        newly, first_res, lam_new = S.count_converged(basis, coeffs, lam_new_dev, limit, bs,
                                                      cfg.tol)
        if lam_new is None:
            lam_new = lam_new_dev.cpu().numpy()
        c = locked + newly
        total_locked = stored + c

        if total_locked >= ne:
            timer.lap("t_step4")
            S.update_in_place(basis, coeffs, v[:, locked:sx])
            lam[locked:sx] = lam_new
            locked = c
            status = "converged"
            if cfg.collect_history:
                theta = select_shift(cfg.shift_mode, lam, locked, store_vals)
                history.append(IterationRecord(it, total_locked, first_res, theta, 0, m, 0,
                                               timer.marks, None, abar_defect))
            break

        compacted = refilled = False
        iter_red = 0
        if cfg.moving and c > 0 and (c >= 2 * bs or c >= sx):
            # window slide (solver.py:325-363)
            if full is None:  # compaction needs the whole spectrum (solver.py:332)
                full = sym_eig_full(dev, abar)
                ops.broadcast(full.values)
                ops.broadcast(full.vectors)
            lam_all = full.values.cpu().numpy()
            # x_all = basis @ full.vectors, in place over the basis (v[:, locked:locked+m]):
            # the emitted pairs [X_locked | x_all[:, :newly]] then already sit right after
            # the store, and the new window x_all[:, newly:] right after them
            S.update_in_place(basis, full.vectors, basis)
            store_vals.append(np.concatenate([lam[:locked], lam_all[:newly]]))
            stored += c
            S_off += c
            v = arena[:, S_off:]
            sx = m - newly
            if sx:
                lam[:sx] = lam_all[newly:]
            locked = 0
            np_, nw = 0, 0
            p_coupling = None
            compacted = True
            c = 0
            if sx < bs:
                add = min(3 * bs, n - stored) - sx
                if add > 0:
                    S.set_random(v[:, sx:sx + add], cfg.seed + 104729 * it)
                    defl = arena[:, :S_off + sx]   # [store, X]: contiguous
                    ro = orth_against(ops, v[:, sx:sx + add], defl, b=Bop, cfg=ocfg)
                    iter_red += ro.reduction_count
                    sx += ro.num_kept
                refilled = True
                if sx <= 0:
                    raise AllDependent("moving window could not be refilled")
        timer.lap("t_step4")

        theta = select_shift(cfg.shift_mode, lam, locked, store_vals)
        cg_rep = None
        if not refilled:
            if compacted:
                bs_eff = max(1, min(bs, ne - stored, sx))
            else:
                bs_eff = max(1, min(bs, ne - stored - c, sx - c))
                phat = S.build_p(coeffs, d, c - locked, bs_eff, ocfg.dependence_tol)
                if phat is None:
                    p_coupling = None
                    cm = coeffs
                else:
                    ap = dev.empty(m, phat.shape[1])
                    D.dgemm(dev, abar, phat, ap)
                    p_coupling = dev.empty(phat.shape[1], phat.shape[1])
                    D.dgemm(dev, phat, ap, p_coupling, ta=True)
                    cm = dev.empty(m, d + phat.shape[1])
                    D.copy(dev, coeffs, cm[:, :d])
                    D.copy(dev, phat, cm[:, d:])
                # [X_new | P_new] = basis [coeffs | phat], written over the basis' head
                S.update_in_place(basis, cm, v[:, locked:locked + cm.shape[1]])
                lam[locked:sx] = lam_new
                locked = c
                np_ = 0 if phat is None else phat.shape[1]
            timer.lap("t_step5")

            # STEP 6: damped inverse power via block CG (solver.py:386-396)
            x_act = v[:, locked:locked + bs_eff]
            w_region = v[:, sx + np_:sx + np_ + bs_eff]
            scale = _h2d(dev, lam[locked:locked + bs_eff] - theta)
            rhs = dev.empty(nloc, bs_eff)
            if Bop is not None:
                ops.spmm(Bop, x_act, rhs)
                D.col_scale(dev, scale, rhs)
            else:
                D.col_scale_copy(dev, scale, x_act, rhs)  # rhs = X (Lambda - theta), one pass
            vals, shift = prob.shifted(theta)
            # initial guess W0 = X read straight from the X block (cg.py:40-45)
            cg_rep = ops.block_cg(vals, shift, rhs, w_region, cfg.cg_max_iters, cfg.cg_rel_tol,
                                  x0=x_act)
            timer.lap("t_step6")

            # STEP 2: W against [store, X, P] (solver.py:398-420): one contiguous range
            defl = arena[:, :S_off + sx + np_]
            try:
                w_out = orth_against(ops, w_region, defl, b=Bop, cfg=ocfg)
                nw = w_out.num_kept
                iter_red += w_out.reduction_count
            except AllDependent:
                nw = 0
            if nw == 0:
                S.set_random(w_region, cfg.seed + 7919 * it)
                try:
                    w_out = orth_against(ops, w_region, defl, b=Bop, cfg=ocfg)
                    nw = w_out.num_kept
                    iter_red += w_out.reduction_count
                except AllDependent:
                    nw = 0
            timer.lap("t_step2")
            if nw and it < cfg.max_gcg_iters:
                pre_timer = _Timer(not det and cfg.collect_history, getattr(dev, "stream", None))
                aw = S.apply_a(v[:, sx + np_:sx + np_ + nw])
                pre_cross = dev.empty(sx - locked + np_ + nw, nw)
                ops.gram(v[:, locked:sx + np_ + nw], aw, pre_cross)

        total_red += iter_red

        basis_defect = None
        if cfg.instrument_orth:
            fb = v[:, :sx + np_ + nw]
            g = dev.empty(fb.shape[1], fb.shape[1])
            ops.gram(fb, S.apply_b(fb), g)
            D.max_abs_diff(dev, g, None, S.scalar)
            basis_defect = float(S.scalar[0].item())

        abar_prev = None if refilled else abar
        if cfg.collect_history:
            rec = IterationRecord(it, total_locked, first_res, theta, 0, m, iter_red,
                                  timer.marks, basis_defect, abar_defect)
            history.append(rec)
            if cg_rep is not None:
                pending_cg.append((rec, cg_rep))

    if pending_cg:  # resolve every CG sweep count with ONE device-to-host read, after the loop
        counts = torch.cat([rep._sweeps.view(-1) for _, rep in pending_cg]).cpu().tolist()
        for (rec, _), cnt in zip(pending_cg, counts):
            rec.cg_iterations = int(cnt)
    # per-step GPU times: the records hold each timer's lazily resolved marks

    # result assembly (solver.py:447-472): store, locked window columns and (when the
    # iterations ran out) Ritz padding are consecutive arena columns
    if store_vals:
        all_vals = np.concatenate(store_vals + [lam[:locked]])
        n_conv = all_vals.shape[0]
        if n_conv < ne:
            extra = min(ne - n_conv, sx - locked)
            all_vals = np.concatenate([all_vals, lam[locked:locked + extra]])
        take = min(ne, all_vals.shape[0])
        values = all_vals[:take].copy()
        vectors = arena[:, :take]
    else:
        n_conv = locked
        values = lam[:ne].copy()
        vectors = v[:, :ne]

    residuals = np.empty(values.shape[0])
    if values.shape[0]:
        vd = torch.from_numpy(values).to(dev.device)
        residuals = S.residuals(vectors, vd)

    # one on-device layout transpose, then a single D2H of an F-order block
    evecs = vectors if cfg.return_device else \
        ops.host_rows(vectors, host_out.take(vectors.shape) if host_out is not None else None)

    return SolverReport(
        status=status,
        eigenvalues=values,
        eigenvectors=evecs,
        num_converged=min(n_conv, ne),
        iterations=iters_run,
        residuals=residuals,
        history=history,
        stagnated=_stagnation_flag(history, cfg.stall_window),
        max_projection_dim=max_m,
        total_reductions=total_red,
        backend=BACKEND_NAME,
        row_range=(ops.row0, ops.row0 + nloc),
    )
