"""Configs 4 and 5 families on the B200: parity at full and mid size.

* BASELINE config 4 (variable-coefficient 7-pt diffusion 128^3, n = 2.1 M, nev = 500,
  moving window, tol 1e-8) at full size: every returned pair meets the north-star
  residual recomputed on the host from the returned vectors, the vectors are
  orthonormal to 1e-9, and the moving-window eigenvalues equal a plain (non-moving)
  device solve to 1e-9 — the reference's own moving == plain acceptance check
  (test_acceptance.py:252-274).  The reference needs ~665 s per GCG iteration for
  this config on 8 cores, so no full reference run exists; the family is pinned to
  the reference by the mid-size golden below and by varcoef10_moving (golden.npz).
* Mid-size members run by the unmodified reference (tests/golden/golden_mid.json,
  make_golden.py --mid): the variable-coefficient operator at 32^3 (nev = 100,
  moving) and config 5's 27-point stencil at 64^3 (nev = 100, moving, tol 1e-7):
  eigenvalues to relative 1e-9, host residuals <= tol.
"""

import json
import os

import numpy as np
import pytest

from paper_2111_06552_b200 import SolverConfig, gcg_solve
from paper_2111_06552_b200 import problems as P

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

HERE = os.path.dirname(os.path.abspath(__file__))
MID = os.path.join(HERE, "golden", "golden_mid.json")


def rel_residuals(a, vals, vecs, chunk=64):
    out = np.empty(vals.shape[0])
    for s in range(0, vals.shape[0], chunk):
        e = min(s + chunk, vals.shape[0])
        x = vecs[:, s:e]
        r = a @ x - x * vals[s:e]
        out[s:e] = np.linalg.norm(r, axis=0) / (np.abs(vals[s:e]) * np.linalg.norm(x, axis=0))
    return out


def _mid(name):
    if not os.path.exists(MID):
        pytest.skip("golden_mid.json not generated")
    ref = json.load(open(MID))
    if name not in ref:
        pytest.skip(f"{name} not in golden_mid.json")
    return ref[name]


@pytest.mark.parametrize("name,build", [
    ("varcoef32_moving", lambda: P.varcoef_diffusion_3d(32, seed=0)),
    ("stencil27_64_moving", lambda: P.stencil27(64)),
])
def test_mid_size_moving_vs_reference(name, build):
    ref = _mid(name)
    a = build()
    kw = dict(ref["kw"])
    rep = gcg_solve(a, None, SolverConfig(**kw, init="normal", residual="relative"))
    want = np.array(ref["eigenvalues"])
    assert rep.status == ref["status"] == "converged"
    assert np.abs(rep.eigenvalues - want).max() <= 1e-9 * np.abs(want).max()
    tol = kw["tol"]
    assert rep.residuals.max() <= tol
    assert rel_residuals(a, rep.eigenvalues, rep.eigenvectors).max() <= 1.01 * tol
    assert rep.max_projection_dim <= ref["max_projection_dim"]
    assert abs(rep.iterations - ref["iterations"]) <= max(4, int(0.15 * ref["iterations"]))


def test_cfg4_full_size_moving_equals_plain():
    pr = P.baseline_problem(4)
    base = dict(num_eigen=500, tol=1e-8, seed=0, init="normal", residual="relative",
                validate=False)
    mov = gcg_solve(pr.a, None, SolverConfig(**base, moving=True))
    assert mov.status == "converged" and mov.num_converged == 500
    assert mov.max_projection_dim <= 5 * 100
    assert mov.residuals.max() <= 1e-8
    v = mov.eigenvectors
    assert rel_residuals(pr.a, mov.eigenvalues, v).max() <= 1.01e-8
    g = v.T @ v
    assert np.abs(g - np.eye(500)).max() <= 1e-9
    assert np.all(np.diff(mov.eigenvalues) >= -1e-12 * mov.eigenvalues[-1])
    del v, g
    plain = gcg_solve(pr.a, None, SolverConfig(**base, moving=False))
    assert plain.status == "converged"
    lam = plain.eigenvalues
    assert np.abs(mov.eigenvalues - lam).max() <= 1e-9 * np.abs(lam).max()
    print(f"cfg4: moving {mov.iterations} iters, plain {plain.iterations} iters, "
          f"max |dlambda|/lambda_max = {np.abs(mov.eigenvalues - lam).max() / lam.max():.2e}")
