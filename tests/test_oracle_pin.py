"""Pin the CPU oracle (oracle/gcg_oracle.py) to the reference's golden vectors.

The golden vectors were produced by the unmodified reference
(tests/golden/make_golden.py).  The oracle restates the reference's numpy
backend operation for operation, so solver runs must agree bit for bit.
"""

import math

import numpy as np
import pytest

from oracle import gcg_oracle as O
from paper_2111_06552_b200 import problems as P
from tests.cases import SOLVER_CASES, problem as _problem


def test_kernel_kats(golden):
    g = golden
    out = O.csr_matvec(g["k_csr_indptr"], g["k_csr_indices"], g["k_csr_data"], g["k_csr_x"])
    # numpy backend is bitwise; the Cython core agrees to atol 1e-13 (test_kernels.py:54)
    assert np.array_equal(out, g["k_csr_out_numpy"])
    if "k_csr_out_compiled" in g:
        assert np.abs(out - g["k_csr_out_compiled"]).max() <= 1e-13
    for det in (0, 1):
        ip = O.inner_product(g["k_ip_x"], g["k_ip_y"], chunk=512, deterministic=bool(det))
        assert np.array_equal(ip, g[f"k_ip_out_numpy_{det}"])
    for i, (al, bt) in enumerate([(0.0, 0.0), (1.0, 0.0), (0.0, 1.0), (2.5, 1.0), (2.5, -0.5)]):
        y = g["k_axpby_y"].copy(order="F")
        O.axpby(al, g["k_axpby_x"], bt, y)
        assert np.array_equal(y, g[f"k_axpby_out_numpy_{i}"])


def test_block_cg(golden):
    g = golden
    a = O.Csr(P.stencil_csr((60,), [(0,), (-1,), (1,)], [2.0, -1.0, -1.0]))
    w, rep = O.block_cg(lambda y: O.shifted_apply(a, None, 0.05, y), g["cg_rhs"], g["cg_x0"], 30, 0.01)
    assert np.array_equal(w, g["cg_w"])
    assert [rep.iterations, rep.converged.sum(), rep.frozen.sum()] == list(g["cg_meta"])
    assert np.array_equal(rep.relative_residuals, g["cg_relres"])


@pytest.mark.parametrize("tag,tol", [("strict", 1e-15), ("default", 1e-10)])
def test_recursive_orth(golden, tag, tol):
    x = golden[f"orth_{tag}_in"].copy(order="F")
    r = O.recursive_orth_svd(x, prm=O.OrthParams(reorth_tol=tol))
    assert [r.num_kept, r.reduction_count] == list(golden[f"orth_{tag}_meta"])
    assert np.array_equal(x, golden[f"orth_{tag}_out"])


def test_recursive_counts_closed_form():
    # m/4 - 1 at three leaf passes, 5 with the adaptive exit (test_orth.py:70-86)
    x = np.asfortranarray(np.random.default_rng(303).uniform(-1, 1, (256, 32)))
    assert O.recursive_orth_svd(x, prm=O.OrthParams(reorth_tol=1e-15)).reduction_count == 7
    x = np.asfortranarray(np.random.default_rng(304).uniform(-1, 1, (256, 32)))
    assert O.recursive_orth_svd(x).reduction_count == 5


def test_orth_against(golden):
    x = golden["oa_in"].copy(order="F")
    r = O.orth_against(x, golden["oa_basis"])
    assert [r.num_kept, r.reduction_count] == list(golden["oa_meta"])
    assert np.array_equal(x, golden["oa_out"])


def test_dense(golden):
    w, v = O.eig_full(golden["m8"])
    assert np.abs(w - golden["m8_values"]).max() < 1e-14
    assert np.abs(v - golden["m8_vectors"]).max() < 1e-13


@pytest.mark.parametrize("name", SOLVER_CASES)
def test_solver_bitwise(golden, golden_meta, name):
    meta = golden_meta["solver"][name]
    a, b = _problem(name)
    kw = dict(meta["kw"])
    if meta["baseline_patch"]:
        kw.update(init="normal", residual="relative")
    rep = O.gcg_solve(a, b, O.OracleConfig(**kw))
    assert rep.status == meta["status"]
    assert rep.iterations == meta["iterations"]
    assert rep.total_reductions == meta["total_reductions"]
    assert [h.num_converged for h in rep.history] == meta["converged"]
    assert [h.cg_iterations for h in rep.history] == meta["cg"]
    assert np.array_equal(rep.eigenvalues, golden[f"s_{name}_values"])
    assert np.array_equal(rep.residuals, golden[f"s_{name}_residuals"])
    if f"s_{name}_vectors" in golden:
        assert np.array_equal(rep.eigenvectors, golden[f"s_{name}_vectors"])


def test_baseline_generators_shapes():
    # nnz pins from SURVEY §8 (verified there by generating the matrices)
    assert P.laplacian_2d(100).nnz == 49_600
    assert P.laplacian_3d(64).nnz == 1_810_432
    a = P.varcoef_diffusion_3d(16)
    assert a.nnz == 16 ** 3 + 2 * 3 * 15 * 16 * 16
    assert abs(a - a.T).max() == 0.0


def test_analytic_eigenvalues_match_dense():
    a = P.laplacian_3d(8).toarray()
    w = np.linalg.eigvalsh(a)[:12]
    assert np.abs(w - P.analytic_eigenvalues(2, 12, scale=8)).max() < 1e-12
    a = P.stencil27(8).toarray()
    w = np.linalg.eigvalsh(a)[:12]
    assert np.abs(w - P.analytic_eigenvalues(5, 12, scale=8)).max() < 1e-12


@pytest.mark.parametrize("tag", ["m8_b2", "m32_b2", "m8_default", "dup_col", "zero_col", "with_b",
                                 "with_x0", "m96_b16"])
def test_modified_block_orth(golden_alg2, tag):
    """Alg. 2 restatement vs the reference run (counts m + m/b - 1, test_orth.py:46-67)."""
    from tests.conftest import ALG2_KW

    g = golden_alg2
    x = g[f"{tag}_in"].copy(order="F")
    x0 = g[f"{tag}_x0"] if f"{tag}_x0" in g else None
    b = None
    if tag == "with_b":
        n = x.shape[0]
        import scipy.sparse

        b = O.Csr(scipy.sparse.diags([np.ones(n - 1), 4.0 * np.ones(n), np.ones(n - 1)], [-1, 0, 1],
                                     format="csr"))
    r = O.modified_block_orth(x, x0=x0, b=b, prm=O.OrthParams(**ALG2_KW[tag]))
    assert [r.num_kept, r.reduction_count] == list(g[f"{tag}_meta"])
    assert r.replaced_indices == list(g[f"{tag}_replaced"])
    assert np.array_equal(x, g[f"{tag}_out"])
