"""Host-side generators for the five BASELINE.json problems.

None of these matrices exists in the reference (its generators are 1-D only,
io.py:257-336), so they are defined here once and shared by the device path,
the CPU oracle and the benchmarks.  All matrices are scipy CSR with int32
indices and float64 values, rows/columns in lexicographic grid order with the
first axis slowest (the row-block / z-slab partition axis of §8(e)).

cfg  problem                                         n            nnz(A)
1    2-D 5-pt Laplacian, 100^2 interior, B = I       10,000       49,600
2    3-D 7-pt Laplacian, 64^3 interior, B = I        262,144      1,810,432
3    P1 FEM stiffness/mass, Kuhn 6-tet split of      493,039      7,246,747 (A and B
     80^3 cube cells, Dirichlet                                   share the 15-pt pattern)
4    var-coef 7-pt diffusion 128^3, harmonic-mean    2,097,152    14,581,760
     faces of exp(N(0,1)) cell coefficients
5    27-pt stencil 256^3 (26, -1), B = I             16,777,216   449,455,096
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse

__all__ = [
    "Problem",
    "stencil_csr",
    "laplacian_2d",
    "laplacian_3d",
    "fem_p1_cube",
    "varcoef_diffusion_3d",
    "stencil27",
    "baseline_problem",
    "analytic_eigenvalues",
]


@dataclass
class Problem:
    name: str
    a: scipy.sparse.csr_matrix
    b: scipy.sparse.csr_matrix | None
    num_eigen: int
    block_size: int | None
    tol: float
    moving: bool
    grid: tuple            # grid shape whose first axis is the partition axis
    description: str


def stencil_csr(shape, offsets, weights):
    """CSR of a constant-or-variable coefficient stencil on a Dirichlet grid.

    ``offsets`` is a list of integer offset tuples; ``weights[t]`` is a scalar
    or an array of length n (per-row coefficient).  Out-of-grid neighbours are
    dropped.  Column indices come out sorted within each row because offsets
    are visited in increasing linear-offset order.
    """
    shape = tuple(int(s) for s in shape)
    nd = len(shape)
    n = int(np.prod(shape))
    strides = [int(np.prod(shape[i + 1:])) for i in range(nd)]
    lin = [sum(o[i] * strides[i] for i in range(nd)) for o in offsets]
    order = np.argsort(lin, kind="stable")
    coords = np.indices(shape, dtype=np.int32).reshape(nd, n)
    rows = np.arange(n, dtype=np.int64)
    colmat = np.empty((n, len(offsets)), dtype=np.int32)
    valmat = np.empty((n, len(offsets)), dtype=np.float64)
    mask = np.empty((n, len(offsets)), dtype=bool)
    for slot, t in enumerate(order):
        off = offsets[t]
        ok = np.ones(n, dtype=bool)
        for ax in range(nd):
            c = coords[ax] + off[ax]
            ok &= (c >= 0) & (c < shape[ax])
        mask[:, slot] = ok
        colmat[:, slot] = (rows + lin[t]).astype(np.int32)
        w = weights[t]
        valmat[:, slot] = w
    del coords
    counts = mask.sum(axis=1)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    cols = colmat[mask]
    vals = valmat[mask]
    del colmat, valmat, mask
    if indptr[-1] < 2**31:
        indptr = indptr.astype(np.int32)
    return scipy.sparse.csr_matrix((vals, cols, indptr), shape=(n, n))


def _axis_offsets(nd):
    offs = []
    for ax in range(nd):
        for s in (-1, 1):
            o = [0] * nd
            o[ax] = s
            offs.append(tuple(o))
    return offs


def laplacian_2d(N):
    """cfg1: I (x) T_N + T_N (x) I, T = tridiag(-1, 2, -1)."""
    offs = [(0, 0)] + _axis_offsets(2)
    return stencil_csr((N, N), offs, [4.0] + [-1.0] * 4)


def laplacian_3d(N):
    """cfg2: T(x)I(x)I + I(x)T(x)I + I(x)I(x)T."""
    offs = [(0, 0, 0)] + _axis_offsets(3)
    return stencil_csr((N, N, N), offs, [6.0] + [-1.0] * 6)


def stencil27(N):
    """cfg5: 27 I - J(x)J(x)J with J = tridiag(1, 1, 1): centre 26, neighbours -1."""
    offs = list(itertools.product((-1, 0, 1), repeat=3))
    w = [26.0 if o == (0, 0, 0) else -1.0 for o in offs]
    return stencil_csr((N, N, N), offs, w)


def varcoef_diffusion_3d(N, seed=0):
    """cfg4: cell-centred 7-pt diffusion with k = exp(g), g ~ N(0,1) per cell.

    Interior face coefficient is the harmonic mean 2 k_a k_b / (k_a + k_b);
    a Dirichlet boundary face adds k_cell to the diagonal.
    """
    rng = np.random.default_rng(seed)
    kc = np.exp(rng.standard_normal((N, N, N)))
    n = N ** 3
    diag = np.zeros((N, N, N))
    offs = [(0, 0, 0)]
    weights = [None]
    for ax in range(3):
        for s in (-1, 1):
            nb = np.roll(kc, -s, axis=ax)
            face = 2.0 * kc * nb / (kc + nb)
            idx = [slice(None)] * 3
            idx[ax] = 0 if s == -1 else N - 1
            bnd = np.zeros((N, N, N), dtype=bool)
            bnd[tuple(idx)] = True
            face = np.where(bnd, 0.0, face)
            diag += face
            diag += np.where(bnd, kc, 0.0)
            o = [0, 0, 0]
            o[ax] = s
            offs.append(tuple(o))
            weights.append(-face.reshape(n))
    weights[0] = diag.reshape(n)
    return stencil_csr((N, N, N), offs, weights)


def _kuhn_local(h):
    """Local P1 stiffness/mass of the six Kuhn tetrahedra of an h-cube."""
    out = []
    for perm in itertools.permutations(range(3)):
        verts = [np.zeros(3, dtype=np.int64)]
        for ax in perm:
            v = verts[-1].copy()
            v[ax] += 1
            verts.append(v)
        p = h * np.array(verts, dtype=np.float64)
        jac = (p[1:] - p[0]).T                       # columns: edge vectors
        vol = abs(np.linalg.det(jac)) / 6.0
        ginv = np.linalg.inv(jac)                    # rows: grads of lambda_1..3
        grads = np.vstack([-ginv.sum(axis=0), ginv])
        k = vol * grads @ grads.T
        m = (vol / 20.0) * (np.ones((4, 4)) + np.eye(4))
        out.append((np.array(verts), k, m))
    return out


def fem_p1_cube(C):
    """cfg3: P1 stiffness A and consistent mass B on the Kuhn-split unit cube.

    C cells per edge, h = 1/C, Dirichlet by keeping the (C-1)^3 interior
    nodes.  A and B are assembled from the same COO pattern, so they share one
    CSR structure (the 15-pt union pattern) — floating assembly residues of
    the stiffness are kept as stored entries.
    """
    h = 1.0 / C
    P = C + 1
    ni = C - 1
    cells = np.indices((C, C, C), dtype=np.int64).reshape(3, -1)
    node_map = np.full(P ** 3, -1, dtype=np.int64)
    g = np.indices((P, P, P), dtype=np.int64).reshape(3, -1)
    interior = ((g >= 1) & (g <= C - 1)).all(axis=0)
    gi = g[:, interior] - 1
    node_map[interior] = (gi[0] * ni + gi[1]) * ni + gi[2]
    rows_l, cols_l, ka_l, mb_l = [], [], [], []
    for verts, kl, ml in _kuhn_local(h):
        gidx = []
        for v in verts:
            c = cells + v[:, None]
            gidx.append(node_map[(c[0] * P + c[1]) * P + c[2]])
        gidx = np.stack(gidx)                        # (4, ncells)
        for a in range(4):
            for b in range(4):
                ok = (gidx[a] >= 0) & (gidx[b] >= 0)
                rows_l.append(gidx[a][ok].astype(np.int32))
                cols_l.append(gidx[b][ok].astype(np.int32))
                cnt = int(ok.sum())
                ka_l.append(np.full(cnt, kl[a, b]))
                mb_l.append(np.full(cnt, ml[a, b]))
    rows = np.concatenate(rows_l)
    cols = np.concatenate(cols_l)
    n = ni ** 3
    a = scipy.sparse.coo_matrix((np.concatenate(ka_l), (rows, cols)), shape=(n, n)).tocsr()
    b = scipy.sparse.coo_matrix((np.concatenate(mb_l), (rows, cols)), shape=(n, n)).tocsr()
    a.sort_indices()
    b.sort_indices()
    assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
    return a, b


_BASELINE = {
    1: dict(name="cfg1-lap2d-100", nev=20, bs=20, tol=1e-8, moving=False),
    2: dict(name="cfg2-lap3d-64", nev=100, bs=None, tol=1e-8, moving=False),
    3: dict(name="cfg3-fem-p1-80", nev=200, bs=None, tol=1e-8, moving=False),
    4: dict(name="cfg4-varcoef-128", nev=500, bs=None, tol=1e-8, moving=True),
    5: dict(name="cfg5-27pt-256", nev=1000, bs=None, tol=1e-7, moving=True),
}


def baseline_problem(cfg, scale=None, build=True):
    """Build BASELINE.json config ``cfg`` (1-based).  ``scale`` overrides the
    grid size (for small parity runs of the same operator family).  With
    ``build=False`` only the metadata is returned (``a`` is None) — for the
    device generators (devgen.py)."""
    spec = _BASELINE[cfg]
    b = None
    a = None
    if cfg == 1:
        N = scale or 100
        grid, desc = (N, N), f"2-D 5-pt Laplacian {N}^2"
        if build:
            a = laplacian_2d(N)
    elif cfg == 2:
        N = scale or 64
        grid, desc = (N, N, N), f"3-D 7-pt Laplacian {N}^3"
        if build:
            a = laplacian_3d(N)
    elif cfg == 3:
        C = scale or 80
        grid, desc = (C - 1,) * 3, f"P1 FEM Kuhn cube {C}^3 cells"
        if build:
            a, b = fem_p1_cube(C)
    elif cfg == 4:
        N = scale or 128
        grid, desc = (N, N, N), f"var-coef 7-pt {N}^3"
        if build:
            a = varcoef_diffusion_3d(N, seed=0)
    elif cfg == 5:
        N = scale or 256
        grid, desc = (N, N, N), f"27-pt stencil {N}^3"
        if build:
            a = stencil27(N)
    else:
        raise KeyError(cfg)
    return Problem(spec["name"] if scale is None else f"{spec['name']}@{scale}", a, b,
                   spec["nev"], spec["bs"], spec["tol"], spec["moving"], grid, desc)


def analytic_eigenvalues(cfg, count, scale=None):
    """Closed-form smallest eigenvalues for cfg 1, 2, 5; None otherwise."""
    if cfg == 1:
        N, nd = scale or 100, 2
        lam1 = 2.0 - 2.0 * np.cos(np.arange(1, N + 1) * math.pi / (N + 1))
    elif cfg == 2:
        N, nd = scale or 64, 3
        lam1 = 2.0 - 2.0 * np.cos(np.arange(1, N + 1) * math.pi / (N + 1))
    elif cfg == 5:
        N = scale or 256
        mu = 1.0 + 2.0 * np.cos(np.arange(1, N + 1) * math.pi / (N + 1))
        # 27 - prod(mu): smallest come from the largest products
        top = np.sort(mu)[::-1][: min(N, 40)]
        prods = np.sort((top[:, None, None] * top[None, :, None] * top[None, None, :]).ravel())[::-1]
        return np.sort(27.0 - prods)[:count]
    else:
        return None
    grids = np.meshgrid(*([lam1[: min(N, 64)]] * nd), indexing="ij")
    tot = sum(grids).ravel()
    return np.sort(tot)[:count]
