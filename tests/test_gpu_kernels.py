"""Kernel parity on the B200: every device op against the CPU oracle / numpy.

Tolerances follow north_star ("SpMM/Gram kernels to 1e-12 relative against the
reference ops") measured normwise and the reference's own
kernel tests (test_kernels.py:43-102).
"""

import os

import numpy as np
import pytest
import scipy.sparse
import torch

from oracle import gcg_oracle as O
from paper_2111_06552_b200 import _lib
from paper_2111_06552_b200 import device as D
from paper_2111_06552_b200 import problems as P
from paper_2111_06552_b200 import refbackend
from paper_2111_06552_b200.operators import DeviceCsr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    return D.default_context()


def rm(dev, a):
    """host array -> row-major device tensor"""
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev.device)


def host(t):
    return t.cpu().numpy()


def rel_err(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


def random_sym_csr(n, density, seed):
    m = scipy.sparse.random(n, n, density=density, random_state=np.random.RandomState(seed))
    m = (m + m.T).tocsr()
    m.sum_duplicates()
    return m


SPMM_CASES = [
    ("lap3d16", lambda: P.laplacian_3d(16)),
    ("27pt10", lambda: P.stencil27(10)),
    ("fem5", lambda: P.fem_p1_cube(5)[1]),
    ("rand300", lambda: random_sym_csr(300, 0.05, 1)),
]


@pytest.mark.parametrize("name,mk", SPMM_CASES)
@pytest.mark.parametrize("k", [1, 3, 7, 20, 40, 100, 200, 300])
def test_spmm_vs_oracle(dev, name, mk, k):
    a = mk()
    A = DeviceCsr.from_scipy(dev, a)
    rng = np.random.default_rng(k)
    x = rng.standard_normal((a.shape[0], k))
    want = O.csr_matvec(a.indptr, a.indices, a.data, np.asfortranarray(x))
    y = dev.empty(a.shape[0], k)
    D.spmm(dev, A, rm(dev, x), y)
    assert rel_err(host(y), want) <= 1e-13


def test_spmm_strided_views_and_epilogue(dev):
    a = P.laplacian_3d(12)
    n = a.shape[0]
    A = DeviceCsr.from_scipy(dev, a)
    rng = np.random.default_rng(3)
    arena = rng.standard_normal((n, 57))
    xa = rm(dev, arena)
    x = xa[:, 5:26]          # odd offset, odd width: scalar path
    z = xa[:, 30:51]
    yin = rng.standard_normal((n, 21))
    out = dev.zeros(n, 40)[:, 3:24]
    dots = dev.empty(21)
    D.spmm(dev, A, x, out, alpha=-1.5, gamma=0.25, Z=z, beta=2.0, Yin=rm(dev, yin), dot_mode=1,
           W=z, dots=dots)
    xs, zs = arena[:, 5:26], arena[:, 30:51]
    want = -1.5 * (a @ xs) + 0.25 * zs + 2.0 * yin
    assert rel_err(host(out), want) <= 1e-13
    assert rel_err(host(dots), (want * zs).sum(0)) <= 1e-12
    dots2 = dev.empty(21)
    D.spmm(dev, A, x, out, dot_mode=2, dots=dots2)
    w2 = a @ xs
    assert rel_err(host(dots2), (w2 * w2).sum(0)) <= 1e-12


@pytest.mark.parametrize("k", [4, 20, 22, 40, 64, 100, 160, 250])
@pytest.mark.parametrize("diag", [True, False])
def test_spmm_self_epilogue(dev, k, diag):
    """The block-CG forms: Z = W = X (diagonal gather reused), 256-bit rows, ragged tails,
    and a pattern without stored diagonal (fallback loads)."""
    a = P.laplacian_3d(9).tocsr()
    if not diag:
        a = (a - scipy.sparse.diags(a.diagonal())).tocsr()
        a.eliminate_zeros()
    n = a.shape[0]
    A = DeviceCsr.from_scipy(dev, a)
    rng = np.random.default_rng(k)
    x = rng.standard_normal((n, k))
    yin = rng.standard_normal((n, k))
    xd = rm(dev, x)
    y = dev.empty(n, k)
    dots = dev.empty(k)
    D.spmm(dev, A, xd, y, alpha=1.0, gamma=-0.7, Z=xd, dot_mode=1, W=xd, dots=dots)
    want = a @ x - 0.7 * x
    assert rel_err(host(y), want) <= 1e-13
    assert rel_err(host(dots), (want * x).sum(0)) <= 1e-12
    D.spmm(dev, A, xd, y, alpha=-1.0, gamma=0.3, Z=xd, beta=1.0, Yin=rm(dev, yin), dot_mode=2,
           dots=dots)
    want = yin - (a @ x) + 0.3 * x
    assert rel_err(host(y), want) <= 1e-13
    assert rel_err(host(dots), (want * want).sum(0)) <= 1e-12


@pytest.mark.parametrize("n,k1,k2", [(1, 1, 1), (23, 4, 3), (5000, 6, 4), (262144, 200, 20),
                                      (100003, 80, 80), (4097, 17, 33), (70000, 120, 7),
                                      # wide 160 x 128 tiles (cfg4 / cfg5 deflation shapes)
                                      (50001, 300, 100), (20000, 900, 100), (30011, 600, 200),
                                      (4099, 161, 65), (8191, 200, 200), (12345, 500, 100)])
def test_gram_vs_numpy(dev, n, k1, k2):
    rng = np.random.default_rng(n + k1)
    x = rng.standard_normal((n, k1))
    y = rng.standard_normal((n, k2))
    g = dev.empty(k1, k2)
    D.gram(dev, rm(dev, x), rm(dev, y), g)
    want = x.T @ y
    scale = np.sqrt((x * x).sum(0)).max() * np.sqrt((y * y).sum(0)).max()
    assert np.abs(host(g) - want).max() / scale <= 1e-13
    g2 = dev.empty(k1, k2)
    D.gram(dev, rm(dev, x), rm(dev, y), g2)
    assert torch.equal(g, g2)  # deterministic: bit-stable run to run (test_kernels.py:74-85)


@pytest.mark.parametrize("off1,k1,off2,k2", [(3, 200, 205, 20), (1, 199, 210, 21), (0, 160, 161, 40),
                                              (5, 96, 101, 96), (2, 17, 40, 7)])
def test_gram_lincomb_odd_column_views(dev, off1, k1, off2, k2):
    """Views at odd columns of an even-ld arena (basis = v[:, locked:], locked odd):
    the bulk-staged kernels copy those rows from one element earlier."""
    n = 40000
    rng = np.random.default_rng(off1 + k1)
    arena = rng.standard_normal((n, 260))
    A = rm(dev, arena)
    x, y = arena[:, off1:off1 + k1], arena[:, off2:off2 + k2]
    g = dev.empty(k1, k2)
    D.gram(dev, A[:, off1:off1 + k1], A[:, off2:off2 + k2], g)
    scale = np.sqrt((x * x).sum(0)).max() * np.sqrt((y * y).sum(0)).max()
    assert np.abs(host(g) - x.T @ y).max() / scale <= 1e-13
    c = rng.standard_normal((k1, k2 + 70))
    out = dev.empty(n, k2 + 70)
    D.lincomb(dev, A[:, off1:off1 + k1], rm(dev, c), out)
    assert rel_err(host(out), x @ c) <= 1e-13
    # in place over the leading columns of the odd-offset view (the [X|P] update)
    d = min(k1, k2 + 70)
    cc = rng.standard_normal((k1, d))
    D.lincomb(dev, A[:, off1:off1 + k1], rm(dev, cc), A[:, off1:off1 + d])
    assert rel_err(host(A[:, off1:off1 + d]), x @ cc) <= 1e-13


def test_gram_strided_out_and_accumulate(dev):
    rng = np.random.default_rng(9)
    x, y = rng.standard_normal((300, 3)), rng.standard_normal((300, 2))
    parent = dev.zeros(6, 5) + 7.5
    view = parent[1:4, 1:3]
    D.gram(dev, rm(dev, x), rm(dev, y), view)
    p = host(parent)
    assert np.abs(p[1:4, 1:3] - x.T @ y).max() < 1e-12
    mask = np.ones_like(p, dtype=bool)
    mask[1:4, 1:3] = False
    assert np.all(p[mask] == 7.5)
    gt = dev.zeros(2, 3)
    D.gram(dev, rm(dev, x), rm(dev, y), gt, transpose_out=True)
    assert np.abs(host(gt) - (x.T @ y).T).max() < 1e-12


@pytest.mark.parametrize("n,m,d", [(1000, 16, 16), (262144, 200, 160), (5000, 7, 3),
                                    (77777, 64, 100), (3000, 300, 20), (30011, 300, 100),
                                    (20001, 600, 200), (5003, 150, 210), (4001, 97, 97),
                                    (9999, 900, 112)])
def test_lincomb_vs_numpy(dev, n, m, d):
    rng = np.random.default_rng(m * d)
    x = rng.standard_normal((n, m))
    c = rng.standard_normal((m, d))
    y0 = rng.standard_normal((n, d))
    y = rm(dev, y0)
    D.lincomb(dev, rm(dev, x), rm(dev, c), y, alpha=-0.5, beta=1.25)
    want = -0.5 * (x @ c) + 1.25 * y0
    assert rel_err(host(y), want) <= 1e-13


@pytest.mark.parametrize("n,m,d,off", [(5000, 200, 180, 0), (3001, 40, 24, 0),
                                        (3001, 40, 20, 7), (777, 64, 64, 0), (5000, 300, 100, 0),
                                        (3001, 400, 200, 0)])
def test_lincomb_in_place(dev, n, m, d, off):
    """[X|P] <- basis [coeffs|phat] written over the basis' own columns (solver step 5)."""
    rng = np.random.default_rng(n + d)
    x = rng.standard_normal((n, m + 3))
    c = rng.standard_normal((m, d))
    v = rm(dev, x)
    D.lincomb(dev, v[:, :m], rm(dev, c), v[:, off:off + d])
    got = host(v)
    assert rel_err(got[:, off:off + d], x[:, :m] @ c) <= 1e-13
    assert np.array_equal(got[:, :off], x[:, :off])
    assert np.array_equal(got[:, off + d:], x[:, off + d:])


def test_lincomb_rejects_cross_row_overlap(dev):
    v = dev.zeros(100, 300)
    cm = dev.zeros(20, 8)
    with pytest.raises(Exception):
        D.lincomb(dev, v[1:, :20], cm, v[:-1, :8])     # Y row i aliases X row i - 1
    with pytest.raises(Exception):
        D.lincomb(dev, v, dev.zeros(300, 260), v[:, :260])  # in place beyond one column tile


def test_axpby_copy_scale_dots(dev):
    rng = np.random.default_rng(5)
    x, y = rng.standard_normal((999, 7)), rng.standard_normal((999, 7))
    for al, bt in [(0.0, 0.0), (1.0, 0.0), (0.0, 1.0), (2.5, 1.0), (2.5, -0.5)]:
        yt = rm(dev, y)
        D.axpby(dev, al, rm(dev, x), bt, yt)
        assert np.abs(host(yt) - (al * x + bt * y)).max() <= 1e-14
    nan = dev.empty(999, 7).fill_(float("nan"))
    D.axpby(dev, 3.0, rm(dev, x), 0.0, nan)  # beta == 0 never reads y
    assert np.array_equal(host(nan), 3.0 * x)
    s = rng.standard_normal(7)
    xt = rm(dev, x)
    D.col_scale(dev, rm(dev, s), xt)
    assert np.abs(host(xt) - x * s).max() <= 1e-15
    out = dev.empty(7)
    D.col_dots(dev, rm(dev, x), rm(dev, y), out)
    assert rel_err(host(out), (x * y).sum(0)) <= 1e-12


@pytest.mark.parametrize("m", [1, 2, 5, 16, 33, 64, 65, 120, 200, 224, 225, 231, 232, 233, 300,
                               400, 500, 777, 1000, 1024, 1025])
def test_syev_vs_lapack(dev, m):
    rng = np.random.default_rng(m)
    a = rng.standard_normal((m, m))
    a = (a + a.T) / 2
    w = dev.empty(m)
    v = dev.empty(m, m)
    D.syev(dev, rm(dev, a), w, v)
    ww, vv = O.eig_full(a)
    assert np.abs(host(w) - ww).max() <= 1e-12 * max(1.0, np.abs(ww).max())
    V = host(v)
    assert np.abs(a @ V - V * host(w)).max() <= 1e-12 * max(1.0, np.abs(ww).max())
    assert np.abs(V.T @ V - np.eye(m)).max() <= 1e-12
    # sign rule of dense.py:63-71 (non-degenerate random spectrum => columns match LAPACK's)
    assert np.abs(V - vv).max() <= 1e-9


def _degenerate(m, seed, kind):
    rng = np.random.default_rng(seed)
    if kind == "lap3d":          # 6^3 Laplacian: eigenvalue multiplicities 1, 3 and 6
        n1 = round(m ** (1 / 3))
        t = 2 * np.eye(n1) - np.eye(n1, k=1) - np.eye(n1, k=-1)
        i = np.eye(n1)
        return np.kron(np.kron(t, i), i) + np.kron(np.kron(i, t), i) + np.kron(np.kron(i, i), t)
    if kind == "clusters":       # rotated spectrum with exact and 1e-9-close clusters, a 0
        w = np.repeat(rng.standard_normal(m // 4), 4)[:m].copy()
        w[: m // 8] += 1e-9 * np.arange(m // 8)
        w[-1] = 0.0
        q, _ = np.linalg.qr(rng.standard_normal((m, m)))
        a = (q * w) @ q.T
        return (a + a.T) / 2
    if kind == "rr":             # Rayleigh-Ritz shape: diag(Ritz values) coupled to a P/W block
        d = (3 * m) // 5 if m > 224 else (160 if m > 160 else m - 10)
        a = np.zeros((m, m))
        a[:d, :d] = np.diag(np.sort(rng.uniform(0.006, 0.3, d)))
        b = 1e-3 * rng.standard_normal((m - d, d))
        c = rng.standard_normal((m - d, m - d))
        a[d:, :d] = b
        a[:d, d:] = b.T
        a[d:, d:] = 0.5 * (c + c.T) + 2 * np.eye(m - d)
        return a
    if kind == "diag":           # already tridiagonal-free: every reflector is the identity
        return np.diag(np.arange(m, dtype=float)[::-1] % 7)
    raise ValueError(kind)


@pytest.mark.parametrize("m,kind", [(216, "lap3d"), (125, "lap3d"), (200, "clusters"),
                                    (96, "clusters"), (200, "rr"), (120, "rr"), (100, "diag"),
                                    (343, "lap3d"), (729, "lap3d"), (1000, "lap3d"),
                                    (400, "clusters"), (1000, "clusters"), (400, "rr"),
                                    (500, "rr"), (1000, "rr"), (500, "diag")])
def test_syev_degenerate_spectra(dev, m, kind):
    """Eigensolver on the structures RR matrices have: exact multiplicities (grid
    symmetries), near-degenerate clusters, an exact zero, the diag + coupling shape.
    Eigenvalues vs LAPACK; vectors by residual, orthonormality and the cluster
    subspaces (any orthonormal basis of a degenerate eigenspace is valid)."""
    a = _degenerate(m, m, kind)
    w = dev.empty(m)
    v = dev.empty(m, m)
    D.syev(dev, rm(dev, a), w, v)
    ww, vv = np.linalg.eigh(a)
    scale = max(1.0, np.abs(ww).max())
    lam, V = host(w), host(v)
    assert np.abs(lam - ww).max() <= 1e-13 * scale * 10
    assert np.abs(a @ V - V * lam).max() <= 1e-13 * scale
    assert np.abs(V.T @ V - np.eye(m)).max() <= 1e-13
    # the span of each cluster matches LAPACK's
    edges = np.flatnonzero(np.diff(ww) > 1e-6 * scale) + 1
    for blk in np.split(np.arange(m), edges):
        s = np.linalg.svd(vv[:, blk].T @ V[:, blk], compute_uv=False)
        assert s.min() >= 1 - 1e-10
    # sign rule of dense.py:63-71: the largest-magnitude entry of every column is positive
    lead = np.abs(V).argmax(axis=0)
    assert (V[lead, np.arange(m)] > 0).all()
    # bit-stable run to run
    w2, v2 = dev.empty(m), dev.empty(m, m)
    D.syev(dev, rm(dev, a), w2, v2)
    assert torch.equal(w, w2) and torch.equal(v, v2)


@pytest.mark.parametrize("m,lo,hi,workers", [(30, 1, 30, 1), (80, 1, 64, 1), (80, 5, 17, 1),
                                             (200, 1, 160, 1), (200, 1, 160, 4), (120, 3, 77, 3),
                                             (16, 2, 9, 1), (400, 1, 320, 1), (500, 1, 300, 1),
                                             (500, 1, 300, 4), (1000, 1, 600, 1),
                                             (1000, 1, 600, 8), (400, 50, 77, 1), (1000, 990, 1000, 1)])
def test_sym_eig_range_vs_lapack(dev, m, lo, hi, workers):
    """sym_eig_range (dense.py:93-117): index ranges (eig.cu bisection + inverse
    iteration of the requested indices), optionally sliced."""
    from paper_2111_06552_b200.dense import split_ranges, sym_eig_range

    rng = np.random.default_rng(m + lo)
    a = rng.standard_normal((m, m))
    a = (a + a.T) / 2
    dec = sym_eig_range(dev, rm(dev, a), lo, hi, workers=workers)
    ww, vv = O.eig_range(a, lo, hi)
    scale = max(1.0, np.abs(ww).max())
    assert np.abs(host(dec.values) - ww).max() <= 1e-12 * scale
    V = host(dec.vectors)
    assert V.shape == (m, hi - lo + 1)
    assert np.abs(a @ V - V * host(dec.values)).max() <= 1e-11 * scale
    assert np.abs(V - vv).max() <= 1e-9  # sign rule, non-degenerate random spectrum
    if workers > 1:
        assert len(split_ranges(lo, hi, workers)) > 1


def test_eigensolver_never_calls_cusolver_up_to_1024(dev):
    """Every BASELINE Rayleigh-Ritz order (m <= 1000, full spectrum and index ranges)
    runs on the library's own kernels: the cuSOLVER call counter does not move."""
    from paper_2111_06552_b200 import _lib
    from paper_2111_06552_b200.dense import sym_eig_full, sym_eig_range

    rng = np.random.default_rng(7)
    n0 = _lib.cusolver_calls()
    for m in (120, 400, 500, 1000):
        a = rng.standard_normal((m, m))
        a = (a + a.T) / 2
        sym_eig_full(dev, rm(dev, a))
        sym_eig_range(dev, rm(dev, a), 1, (3 * m) // 5)
    torch.cuda.synchronize()
    assert _lib.cusolver_calls() == n0
    a = rng.standard_normal((1025, 1025))
    sym_eig_full(dev, rm(dev, (a + a.T) / 2))  # beyond 1024: cuSOLVER syevd
    assert _lib.cusolver_calls() == n0 + 1


_GRID_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2111_06552_b200 import device as D
dev = D.default_context()
for m in (3, 4, 9, 17, 65, 120, 200, 224):
    rng = np.random.default_rng(m)
    a = rng.standard_normal((m, m)); a = (a + a.T) / 2
    w = dev.empty(m); v = dev.empty(m, m)
    D.syev(dev, torch.from_numpy(a).to(dev.device), w, v)
    ww = np.linalg.eigvalsh(a); lam = w.cpu().numpy(); V = v.cpu().numpy()
    s = max(1.0, np.abs(ww).max())
    assert np.abs(lam - ww).max() <= 1e-12 * s, m
    assert np.abs(a @ V - V * lam).max() <= 1e-12 * s, m
    assert np.abs(V.T @ V - np.eye(m)).max() <= 1e-12, m
print("grid-ok")
"""


@pytest.mark.parametrize("mode", ["g", "c", "o"])
def test_tridiagonalisation_variants_small_orders(mode):
    """Each tridiagonalisation variant forced below its default range (GCG_TRIMODE:
    g = co-resident grid, c = one cluster, o = one CTA), including the one- and
    two-row-per-CTA edge cases m = 3, 4, 9, agrees with LAPACK."""
    import subprocess
    import sys

    env = dict(os.environ, GCG_TRIMODE=mode, GCG_SYEV="tri")
    r = subprocess.run([sys.executable, "-c", _GRID_SCRIPT], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "grid-ok" in r.stdout, r.stdout + r.stderr


def test_syev_golden_m8(dev, golden):
    w = dev.empty(8)
    v = dev.empty(8, 8)
    D.syev(dev, rm(dev, golden["m8"]), w, v)
    assert np.abs(host(w) - golden["m8_values"]).max() < 1e-13
    assert np.abs(host(v) - golden["m8_vectors"]).max() < 1e-12


@pytest.mark.parametrize("w,rank", [(6, 6), (16, 16), (16, 11), (40, 40), (100, 100), (90, 60)])
def test_svqb_prepare(dev, w, rank):
    rng = np.random.default_rng(w + rank)
    blk = rng.standard_normal((500, rank)) @ rng.standard_normal((rank, w))
    g = blk.T @ blk
    q = dev.empty(w, w)
    st = dev.empty(4)
    D.svqb_prepare(dev, rm(dev, g), 1e-10, q, st)
    defect, nbad, wmax = host(st)[:3]
    ww, vv = O.gram_eig((g + g.T) / 2)
    floor = 1e-10 * max(ww.max(), 0.0)
    assert int(nbad) == int(np.searchsorted(ww, floor, side="right")) == w - rank
    assert abs(defect - np.abs(g - np.eye(w)).max()) <= 1e-12 * np.abs(g).max()
    kept = w - int(nbad)
    Q = host(q)[:, :kept]
    nb = blk @ Q
    assert np.abs(nb.T @ nb - np.eye(kept)).max() <= 1e-8


def test_block_cg_vs_oracle(dev, golden):
    a = P.stencil_csr((60,), [(0,), (-1,), (1,)], [2.0, -1.0, -1.0])
    from paper_2111_06552_b200.cg import block_cg
    from paper_2111_06552_b200.operators import DeviceProblem

    prob = DeviceProblem(dev, a)
    x = rm(dev, golden["cg_x0"])
    _, rep = block_cg(dev, prob, 0.05, rm(dev, golden["cg_rhs"]), x, 30, 0.01)
    assert rep.iterations == int(golden["cg_meta"][0])
    assert rep.converged.sum() == int(golden["cg_meta"][1])
    assert rel_err(host(x), golden["cg_w"]) <= 1e-10
    assert np.abs(rep.relative_residuals - golden["cg_relres"]).max() <= 1e-10


@pytest.mark.parametrize("shape,k", [
    ((13, 11, 9), 100),   # one row per warp step: the staged (bulk-copied p/q/x) sweep
    ((13, 11, 9), 72),    # staged, 18 lanes per row
    ((15, 15, 15), 20),   # six rows per warp step, bulk r-update with a ragged last stage
    ((17, 9), 21),        # odd k: runs padded to 24 columns (zero right-hand sides)
    ((15, 15, 15), 19),   # padded to 20
    ((9, 9, 9), 5),       # padded to 8
    ((9, 9, 9), 3),       # k <= 4: unpadded, scalar gathers and the register-streamed r-update
    ((7, 7, 7), 256),     # widest single pass
    ((41, 37), 64),
])
def test_block_cg_shapes_vs_oracle(dev, shape, k):
    """The fused sweep variants (prefetching / staged) and both r-update kernels against the
    oracle's cg.py restatement: sweep counts, per-column flags and iterates (cg.py:33-99)."""
    from paper_2111_06552_b200.cg import block_cg
    from paper_2111_06552_b200.operators import DeviceProblem

    offs = [(0,) * len(shape)] + [tuple(s * (i == ax) for i in range(len(shape)))
                                  for ax in range(len(shape)) for s in (-1, 1)]
    a = P.stencil_csr(shape, offs, [2.0 * len(shape)] + [-1.0] * (2 * len(shape)))
    n = a.shape[0]
    rng = np.random.default_rng(k)
    rhs = rng.standard_normal((n, k))
    rhs[:, 1] = 0.0                               # zero right-hand side: converged at sweep 0
    rhs[:, 2] *= 1e-3
    x0 = 0.1 * rng.standard_normal((n, k))
    x0[:, 1] = 0.0
    theta = -0.3
    oa = O.Csr(a)
    want, wrep = O.block_cg(lambda y: O.shifted_apply(oa, None, theta, y), rhs, x0, 12, 0.05)
    x = rm(dev, x0)
    _, rep = block_cg(dev, DeviceProblem(dev, a), theta, rm(dev, rhs), x, 12, 0.05)
    assert rep.iterations == wrep.iterations
    assert np.array_equal(np.asarray(rep.converged, bool), np.asarray(wrep.converged, bool))
    assert rel_err(host(x), want) <= 1e-10
    assert np.abs(rep.relative_residuals - wrep.relative_residuals).max() <= 1e-10


def test_block_cg_semantics(dev):
    """test_cg.py cases: zero-rhs column, indefinite freeze, iteration cap."""
    from paper_2111_06552_b200.cg import block_cg
    from paper_2111_06552_b200.operators import DeviceProblem

    prob = DeviceProblem(dev, scipy.sparse.diags([1.0, -1.0]).tocsr())
    rhs = np.zeros((2, 2))
    rhs[0, 0] = rhs[1, 1] = 1.0
    x = dev.zeros(2, 2)
    _, rep = block_cg(dev, prob, 0.0, rm(dev, rhs), x, 10, 1e-12)
    assert rep.converged[0] and rep.frozen[1] and not rep.converged[1]
    assert np.isfinite(host(x)).all()
    prob = DeviceProblem(dev, scipy.sparse.diags([1.0, 2.0, 3.0]).tocsr())
    rhs = np.zeros((3, 2))
    rhs[:, 1] = [1.0, 0.0, 0.0]
    x = dev.zeros(3, 2)
    _, rep = block_cg(dev, prob, 0.0, rm(dev, rhs), x, 10, 1e-12)
    assert rep.converged.all() and np.all(host(x)[:, 0] == 0.0)
    assert rep.relative_residuals[0] == 0.0
    t = P.stencil_csr((100,), [(0,), (-1,), (1,)], [2.0, -1.0, -1.0])
    prob = DeviceProblem(dev, t)
    rhs = np.zeros((100, 1))
    rhs[0, 0] = 1.0
    x = dev.zeros(100, 1)
    _, rep = block_cg(dev, prob, 0.0, rm(dev, rhs), x, 3, 1e-14)
    assert rep.iterations == 3 and not rep.converged.any()


def test_reference_ffi_tier_golden(golden):
    """gcgeig_* host-buffer entry points against the reference's KAT outputs."""
    g = golden
    out = np.zeros((120, 7), order="F")
    refbackend.csr_matvec(g["k_csr_indptr"], g["k_csr_indices"], g["k_csr_data"], g["k_csr_x"], out)
    assert np.abs(out - g["k_csr_out_numpy"]).max() <= 1e-13
    for det in (0, 1):
        ip = np.empty((6, 4), order="F")
        refbackend.inner_product(g["k_ip_x"], g["k_ip_y"], ip, 512, bool(det))
        assert np.abs(ip - g[f"k_ip_out_numpy_{det}"]).max() <= 1e-11
    for i, (al, bt) in enumerate([(0.0, 0.0), (1.0, 0.0), (0.0, 1.0), (2.5, 1.0), (2.5, -0.5)]):
        y = g["k_axpby_y"].copy(order="F")
        refbackend.axpby(al, g["k_axpby_x"], bt, y)
        assert np.abs(y - g[f"k_axpby_out_numpy_{i}"]).max() <= 1e-14
    # strided out view, guard bytes untouched (test_multivec.py:129-139)
    parent = np.full((8, 7), 7.5, order="F")
    view = parent[1:7, 2:6]
    refbackend.inner_product(g["k_ip_x"], g["k_ip_y"], view, 8, True)
    assert np.abs(view - g["k_ip_out_numpy_0"]).max() <= 1e-11
    mask = np.ones_like(parent, dtype=bool)
    mask[1:7, 2:6] = False
    assert np.all(parent[mask] == 7.5)


def test_launch_counter_moves(dev):
    before = _lib.launch_count()
    y = dev.empty(10, 2)
    D.fill(dev, y, 1.0)
    assert _lib.launch_count() > before


# -- SELL-C-sigma ---------------------------------------------------------------


def _ragged(n, seed):
    """Rows of very different lengths (0 .. 60 nonzeros), symmetric."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, 30, n)
    lens[::17] = 0
    rows = np.repeat(np.arange(n), lens)
    cols = rng.integers(0, n, rows.size)
    m = scipy.sparse.csr_matrix((rng.standard_normal(rows.size), (rows, cols)), shape=(n, n))
    m = (m + m.T).tocsr()
    m.sum_duplicates()
    return m


SELL_CASES = [
    ("lap3d13", lambda: P.laplacian_3d(13)),          # n = 2197: ragged last slice
    ("27pt10", lambda: P.stencil27(10)),
    ("fem5", lambda: P.fem_p1_cube(5)[1]),
    ("ragged", lambda: _ragged(3000, 4)),
]


@pytest.mark.parametrize("name,mk", SELL_CASES)
@pytest.mark.parametrize("sigma", [1, 1024])
@pytest.mark.parametrize("k", [1, 7, 20, 40, 300])
def test_spmm_sell_equals_csr(dev, name, mk, sigma, k):
    """gcg_spmm_sell (rows length-sorted or not) == gcg_spmm_csr, incl. the fused
    shift / axpby / dot epilogues, and == the oracle."""
    from paper_2111_06552_b200.operators import DeviceSell

    a = mk()
    n = a.shape[0]
    A = DeviceCsr.from_scipy(dev, a)
    S = DeviceSell(A, sigma=sigma)
    assert S.nnz_padded >= a.nnz
    rng = np.random.default_rng(k + sigma)
    x = rng.standard_normal((n, k))
    yin = rng.standard_normal((n, k))
    xd, yd = rm(dev, x), rm(dev, yin)
    for kw in (dict(), dict(alpha=-1.0, gamma=0.3, Z=xd, beta=1.0, Yin=yd, dot_mode=2),
               dict(gamma=-0.7, Z=xd, dot_mode=1, W=xd)):
        y1, y2 = dev.empty(n, k), dev.empty(n, k)
        d1, d2 = dev.empty(k), dev.empty(k)
        extra = dict(dots=d1) if "dot_mode" in kw else {}
        S.apply(xd, y1, **kw, **extra)
        D.spmm(dev, A, xd, y2, **kw, **(dict(dots=d2) if "dot_mode" in kw else {}))
        assert torch.equal(y1, y2), name
        want = kw.get("alpha", 1.0) * (a @ x) + kw.get("gamma", 0.0) * x
        if "Yin" in kw:
            want = want + yin
        assert rel_err(host(y1), want) <= 1e-13
        if "dot_mode" in kw:
            ref = (want * want).sum(0) if kw["dot_mode"] == 2 else (want * x).sum(0)
            assert rel_err(host(d1), ref) <= 1e-12


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (200, 20, 200), (20, 20, 200), (200, 200, 200),
                                   (17, 33, 300), (40, 13, 129), (5, 7, 128), (300, 40, 1000)])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_dgemm_small_vs_numpy(dev, M, N, K, ta, tb):
    """Small dense GEMM (momentum block, P coupling): every output one fma chain over k."""
    rng = np.random.default_rng(M * 1000 + N * 10 + K)
    a = rng.standard_normal((K, M) if ta else (M, K))
    b = rng.standard_normal((N, K) if tb else (K, N))
    c0 = rng.standard_normal((M, N))
    want = 0.75 * ((a.T if ta else a) @ (b.T if tb else b)) - 0.5 * c0
    cm = rm(dev, c0)
    D.dgemm(dev, rm(dev, a), rm(dev, b), cm, ta=ta, tb=tb, alpha=0.75, beta=-0.5)
    assert rel_err(host(cm), want) <= 1e-13
    # strided views (leading dimension > columns), beta = 0 never reads C
    big = rm(dev, np.full((M, N + 5), np.nan))
    D.dgemm(dev, rm(dev, a), rm(dev, b), big[:, 2:2 + N], ta=ta, tb=tb)
    assert rel_err(host(big[:, 2:2 + N]), (a.T if ta else a) @ (b.T if tb else b)) <= 1e-13


# Tile shapes added late in round 1 (160 x 48 Gram for k1 > 128, k2 in (32, 48];
# 112-wide Gram / LinComb tiles for k2, d in (96, 112]) on ODD leading dimensions —
# an arena of width sx + 2 bs is odd whenever nev is odd, and then the staged kernels
# take their non-bulk (VEC16 / scalar cp.async) paths.
ODD_LD_SHAPES = [(300, 40, 0), (140, 33, 0), (600, 100, 0), (200, 97, 112), (40, 8, 100)]


def _odd_ld_case(dev, k1, k2, d, seed):
    n = 20011
    ld = k1 + max(k2, d) + 3
    ld += 1 - ld % 2  # odd
    rng = np.random.default_rng(seed)
    arena = rng.standard_normal((n, ld))
    A = rm(dev, arena)
    x, y = arena[:, :k1], arena[:, k1:k1 + k2]
    g = dev.empty(k1, k2)
    D.gram(dev, A[:, :k1], A[:, k1:k1 + k2], g)
    scale = np.sqrt((x * x).sum(0)).max() * np.sqrt((y * y).sum(0)).max()
    assert np.abs(host(g) - x.T @ y).max() / scale <= 1e-13
    if d:
        c = rng.standard_normal((k1, d))
        out = dev.empty(n, d)
        D.lincomb(dev, A[:, :k1], rm(dev, c), out)
        assert rel_err(host(out), x @ c) <= 1e-13
        dd = min(k1, d)
        D.lincomb(dev, A[:, 1:1 + k1], rm(dev, c[:, :dd]), A[:, 1:1 + dd])  # odd offset, in place
        assert rel_err(host(A[:, 1:1 + dd]), arena[:, 1:1 + k1] @ c[:, :dd]) <= 1e-13


@pytest.mark.parametrize("k1,k2,d", ODD_LD_SHAPES)
def test_gram_lincomb_new_tiles_odd_ld(dev, k1, k2, d):
    _odd_ld_case(dev, k1, k2, d, k1 * 7 + k2)


def test_gram_lincomb_new_tiles_odd_ld_without_bulk_copies():
    """Same shapes with GCG_GRAM_BULK=0 / GCG_LINCOMB_BULK=0 (switches read once per
    process, so in a subprocess): the cp.async staging paths."""
    import subprocess
    import sys

    code = ("import tests.test_gpu_kernels as T\n"
            "from paper_2111_06552_b200 import device as D\n"
            "dev = D.default_context()\n"
            "for i, (k1, k2, d) in enumerate(T.ODD_LD_SHAPES):\n"
            "    T._odd_ld_case(dev, k1, k2, d, 100 + i)\n"
            "print('ok')\n")
    env = dict(os.environ, GCG_GRAM_BULK="0", GCG_LINCOMB_BULK="0")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=ROOT, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stdout[-2000:] + out.stderr[-3000:]
