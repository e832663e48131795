"""Parity of the device paths against the reference where round 1 only compared the
device with itself.

* Alg. 3 (recursive_orth_svd / orth_against, orth.py:124-226, 339-372) on the
  reference's own outputs (tests/golden/golden.npz orth_* / oa_*, produced by the
  unmodified reference): kept columns and reduction counts exactly, the block to
  1e-12, Gram defect <= 1e-9 (test_orth.py:46-107) — for the native C++ decision
  loop and for the Python control flow.
* The MultiVec* surface (multivec.py:62-112 + LinearComb) against the CPU oracle.
* BASELINE configs 1 and 2: eigenvectors against the analytic separable-sine
  eigenspaces, per eigenvalue cluster (north-star subspace angle <= 1e-6); the
  cluster cut by nev (cfg2: lambda_100 = lambda_101) is checked for containment in
  the full cluster eigenspace.
"""

import itertools

import numpy as np
import pytest
import torch

from oracle import gcg_oracle as O
from paper_2111_06552_b200 import OrthConfig, SolverConfig, gcg_solve
from paper_2111_06552_b200 import device as D
from paper_2111_06552_b200 import multivec as MV
from paper_2111_06552_b200 import orth as OR
from paper_2111_06552_b200 import problems as P
from paper_2111_06552_b200.operators import DeviceCsr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    return D.default_context()


def _gram_defect(x, b=None):
    bx = x if b is None else b @ x
    return float(np.abs(x.T @ bx - np.eye(x.shape[1])).max())


def _span_sin(got, want, b=None):
    """sin of the largest principal angle between span(got) and span(want), both
    B-orthonormal: ||(I - W W'B) G||_B."""
    bg = got if b is None else b @ got
    y = got - want @ (want.T @ bg)
    by = y if b is None else b @ y
    return float(np.sqrt(max(0.0, np.linalg.eigvalsh(y.T @ by).max())))


def _blocks_match(got, want, b=None, tol=1e-12, leaf=16):
    """Equal blocks where the SVQB output is determined; equal spans where it is not.

    A repeat SVQB pass (orth.py:168-175) factors a Gram matrix that is already I to
    ~1e-15: its eigenvectors — hence the output basis of that leaf — are an arbitrary
    rotation inside the (numerically) degenerate eigenspace, so two correct
    implementations agree on the leaf's span (and on everything the solver uses: the
    iteration depends only on span(V)), not on its columns.  Leaf by
    leaf, spans of the nested prefixes must agree."""
    k = got.shape[1]
    if np.abs(got - want).max() <= tol:
        return True
    for j in sorted(set(list(range(leaf, k, leaf)) + [k])):
        if _span_sin(got[:, :j], want[:, :j], b) > 1e3 * tol:
            return False
    return True


@pytest.fixture(params=["native", "python"])
def driver(request):
    saved = OR._NATIVE
    OR._NATIVE = request.param == "native"
    yield request.param
    OR._NATIVE = saved


@pytest.mark.parametrize("tag,tol", [("strict", 1e-15), ("default", 1e-10)])
def test_recursive_orth_matches_reference(dev, golden, driver, tag, tol):
    """test_orth.py:70-86: 7 reductions at reorth_tol 1e-15, 5 at the default."""
    x = torch.from_numpy(np.ascontiguousarray(golden[f"orth_{tag}_in"])).to(dev.device)
    out = OR.recursive_orth_svd(dev, x, cfg=OrthConfig(reorth_tol=tol))
    kept, red = (int(v) for v in golden[f"orth_{tag}_meta"])
    assert (out.num_kept, out.reduction_count) == (kept, red) == (32, 7 if tag == "strict" else 5)
    assert out.replaced_indices == []
    got = x.cpu().numpy()
    want = golden[f"orth_{tag}_out"]
    if tag == "default":  # every leaf stops after its second Gram check: columns determined
        assert np.abs(got - want).max() <= 1e-12
    assert _blocks_match(got, want)
    assert _gram_defect(got) <= 1e-12 if tag == "strict" else _gram_defect(got) <= 1e-10


def test_orth_against_matches_reference(dev, golden, driver):
    """orth_against (orth.py:339-372) of a block with one spanned column."""
    x = torch.from_numpy(np.ascontiguousarray(golden["oa_in"])).to(dev.device)
    basis = torch.from_numpy(np.ascontiguousarray(golden["oa_basis"])).to(dev.device)
    out = OR.orth_against(dev, x, basis)
    kept, red = (int(v) for v in golden["oa_meta"])
    assert (out.num_kept, out.reduction_count) == (kept, red)
    got = x.cpu().numpy()[:, :kept]
    want = golden["oa_out"][:, :kept]
    assert np.abs(got - want).max() <= 1e-12
    assert _gram_defect(got) <= 1e-9
    assert np.abs(golden["oa_basis"].T @ got).max() <= 1e-9


@pytest.mark.parametrize("seed", range(20))
def test_recursive_orth_property_sweep(dev, driver, seed):
    """test_orth.py:121-136 (many seeds): full rank kept, defect <= 1e-9, span kept;
    the decisions and counts equal the oracle's (pinned to the reference)."""
    rng = np.random.default_rng(5000 + seed)
    n = int(rng.integers(10, 90))
    m = int(rng.integers(2, min(n, 24) + 1))
    xin = rng.uniform(-1, 1, (n, m))
    x = torch.from_numpy(xin.copy()).to(dev.device)
    out = OR.recursive_orth_svd(dev, x)
    ref = np.asfortranarray(xin.copy())
    rr = O.recursive_orth_svd(ref)
    assert (out.num_kept, out.reduction_count) == (rr.num_kept, rr.reduction_count) == \
        (m, rr.reduction_count)
    got = x.cpu().numpy()
    assert _gram_defect(got) <= 1e-9
    proj = got @ (got.T @ xin)
    assert np.abs(xin - proj).max() / np.abs(xin).max() <= 1e-8
    assert np.abs(got - ref).max() <= 1e-10


@pytest.mark.parametrize("use_b", [False, True])
def test_recursive_orth_dependent_and_b(dev, driver, use_b):
    """Rank deficiency (pull_rear, orth.py:95-108) and a B inner product: the same
    replaced slots, counts and block as the oracle."""
    import scipy.sparse

    rng = np.random.default_rng(77)
    n, m = 200, 24
    xin = rng.uniform(-1, 1, (n, m))
    xin[:, 5] = xin[:, 2]
    xin[:, 17] = 0.0
    bs = scipy.sparse.diags([np.ones(n - 1), 4.0 * np.ones(n), np.ones(n - 1)], [-1, 0, 1],
                            format="csr") if use_b else None
    b = DeviceCsr.from_scipy(dev, bs) if use_b else None
    x = torch.from_numpy(xin.copy()).to(dev.device)
    out = OR.recursive_orth_svd(dev, x, b=b)
    ref = np.asfortranarray(xin.copy())
    rr = O.recursive_orth_svd(ref, b=O.Csr(bs) if use_b else None)
    assert (out.num_kept, out.reduction_count, out.replaced_indices) == \
        (rr.num_kept, rr.reduction_count, list(rr.replaced_indices))
    k = out.num_kept
    got = x.cpu().numpy()[:, :k]
    assert _blocks_match(got, ref[:, :k], bs, tol=1e-12)
    assert _gram_defect(got, bs) <= 1e-9


# ---- MultiVec* surface (multivec.py:62-112, LinearComb) vs the oracle -------------------


def test_multivec_surface_vs_oracle(dev):
    rng = np.random.default_rng(42)
    a = P.laplacian_3d(14)  # n = 2744
    n = a.shape[0]
    A = DeviceCsr.from_scipy(dev, a)
    xh = rng.standard_normal((n, 12))
    yh = rng.standard_normal((n, 9))
    x = torch.from_numpy(xh).to(dev.device)
    y = torch.from_numpy(yh).to(dev.device)

    # MatDotMultiVec on a column range
    ax = MV.mat_dot_mv(A, x, cols=(2, 9)).cpu().numpy()
    want = O.csr_matvec(a.indptr, a.indices, a.data, np.asfortranarray(xh[:, 2:9]))
    assert np.abs(ax - want).max() <= 1e-12 * np.abs(want).max()

    # MultiVecInnerProd with B, column ranges and a strided out view
    big = dev.zeros(20, 30)
    view = big[3:10, 5:26:4]  # 7 x 6, non-unit column stride
    MV.mv_inner_prod(x, y, b=A, out=view, x_cols=(1, 8), y_cols=(3, 9))
    by = a @ yh[:, 3:9]
    want = O.inner_product(np.asfortranarray(xh[:, 1:8]), np.asfortranarray(by))
    scale = np.linalg.norm(xh[:, 1:8], axis=0).max() * np.linalg.norm(by, axis=0).max()
    assert np.abs(view.cpu().numpy() - want).max() <= 1e-13 * scale
    untouched = big.cpu().numpy().copy()
    untouched[3:10, 5:26:4] = 0.0
    assert not untouched.any()  # only the viewed entries are written

    # MultiVecAxpby on column ranges, beta = 0 never reads y
    for al, be in [(0.0, 0.0), (1.0, 0.0), (0.0, 1.0), (2.5, 1.0), (2.5, -0.5)]:
        yy = y.clone()
        if be == 0.0:
            yy[:, 2:6] = float("nan")
        MV.mv_axpby(al, x, be, yy, x_cols=(4, 8), y_cols=(2, 6))
        ref = np.asfortranarray(yh[:, 2:6].copy())
        O.axpby(al, np.asfortranarray(xh[:, 4:8]), be, ref)
        got = yy.cpu().numpy()
        assert np.abs(got[:, 2:6] - ref).max() <= 1e-14 * max(1.0, np.abs(ref).max())
        assert np.array_equal(got[:, :2], yh[:, :2]) and np.array_equal(got[:, 6:], yh[:, 6:])

    # MultiVecLinearComb: out = alpha X C + beta out
    ch = rng.standard_normal((12, 7))
    cdev = torch.from_numpy(ch).to(dev.device)
    out = torch.from_numpy(yh[:, :7].copy()).to(dev.device)
    MV.mv_linear_comb(x, cdev, out=out, alpha=-1.5, beta=0.5)
    want = -1.5 * xh @ ch + 0.5 * yh[:, :7]
    assert np.abs(out.cpu().numpy() - want).max() <= 1e-13 * np.abs(want).max()


# ---- analytic eigenspaces of BASELINE configs 1 and 2 -----------------------------------


def _sine_modes(N):
    i = np.arange(1, N + 1)
    lam = 2.0 - 2.0 * np.cos(i * np.pi / (N + 1))
    vec = np.sqrt(2.0 / (N + 1)) * np.sin(np.outer(np.arange(1, N + 1), i) * np.pi / (N + 1))
    return lam, vec  # vec[:, a] is mode a+1 (unit norm)


def _analytic_clusters(dims, N, count, gap=1e-8):
    """Eigenvalue clusters of the separable Dirichlet Laplacian (sorted), covering at least
    the `count` smallest eigenvalues, the last cluster complete."""
    lam1, _ = _sine_modes(N)
    modes = sorted(itertools.product(range(12), repeat=dims), key=lambda t: sum(lam1[list(t)]))
    vals = np.array([sum(lam1[list(t)]) for t in modes])
    clusters, j = [], 0
    while j < len(vals) and (not clusters or clusters[-1][0] < count):
        e = j + 1
        while e < len(vals) and vals[e] - vals[e - 1] <= gap * vals[e]:
            e += 1
        clusters.append((j, e))
        j = e
    return vals, modes, clusters


def _mode_vectors(dims, N, modes):
    _, v1 = _sine_modes(N)
    cols = []
    for t in modes:
        u = v1[:, t[0]]
        for a in t[1:]:
            u = np.multiply.outer(u, v1[:, a])
        cols.append(u.ravel())
    return np.stack(cols, axis=1)


def _check_eigenspaces(dims, N, rep, nev):
    vals, modes, clusters = _analytic_clusters(dims, N, nev)
    w = rep.eigenvectors
    worst = 0.0
    for j, e in clusters:
        if j >= nev:
            break
        u = _mode_vectors(dims, N, modes[j:e])       # full exact cluster eigenspace
        wj = w[:, j:min(e, nev)]                     # returned members (maybe cut by nev)
        assert np.abs(rep.eigenvalues[j:min(e, nev)] - vals[j:min(e, nev)]).max() <= \
            1e-9 * vals[-1]
        y = wj - u @ (u.T @ wj)                      # component outside the eigenspace
        sin = float(np.sqrt(max(0.0, np.linalg.eigvalsh(y.T @ y).max())))
        worst = max(worst, sin)
    return worst


def test_cfg1_eigenvectors_vs_analytic_eigenspaces():
    pr = P.baseline_problem(1)
    rep = gcg_solve(pr.a, None, SolverConfig(num_eigen=20, block_size=20, tol=1e-8, seed=0,
                                             init="normal", residual="relative"))
    assert rep.status == "converged"
    assert _check_eigenspaces(2, 100, rep, 20) <= 1e-6


@pytest.mark.slow
def test_cfg2_eigenvectors_vs_analytic_eigenspaces():
    pr = P.baseline_problem(2)
    rep = gcg_solve(pr.a, None, SolverConfig(num_eigen=100, tol=1e-8, seed=0, init="normal",
                                             residual="relative"))
    assert rep.status == "converged"
    worst = _check_eigenspaces(3, 64, rep, 100)
    print(f"cfg2 worst cluster subspace sin = {worst:.2e}")
    assert worst <= 1e-6
