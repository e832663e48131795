"""Generate golden vectors by running the UNMODIFIED reference (gcgeig).

Run in the build container, where the reference is available — either built
into oracle/_ref (oracle/build_ref.sh) or importable from /root/reference:

    python tests/golden/make_golden.py            # small cases -> golden.npz (+ Alg. 2)
    python tests/golden/make_golden.py --alg2     # Alg. 2 cases only -> golden_alg2.npz
    python tests/golden/make_golden.py --cfg 2    # BASELINE config 2 (~8 min)
    python tests/golden/make_golden.py --cfg 3    # BASELINE config 3 (~1-2 h)
    python tests/golden/make_golden.py --mid      # cfg4/cfg5-family mid-size moving runs

The outputs are committed; the GPU box (which has no /root/reference) only
reads them.  Parity cases follow SURVEY.md §8(c): the reference's own KAT
shapes (test_kernels.py, test_cg.py, test_orth.py, test_dense.py) plus solver
runs on small members of the BASELINE operator families.  For BASELINE-style
runs the reference is monkeypatched exactly as BASELINE.md §3 prescribes:
`solver.mv_set_random` draws N(0,1) and `solver._rel_residual` is the
north-star criterion ||Ax - lam Bx|| / (|lam| ||Bx||).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np
import scipy.sparse

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2111_06552_b200 import problems as P  # noqa: E402

gcgeig = oracle.load_reference()
if gcgeig is None:  # fall back to the read-only source tree (numpy backend only)
    sys.path.insert(0, "/root/reference/pkg/src")
    import gcgeig  # noqa: E402

from gcgeig import SolverConfig, gcg_solve  # noqa: E402
from gcgeig import _kernels as K  # noqa: E402
from gcgeig import orth as R  # noqa: E402
from gcgeig import solver as S  # noqa: E402
from gcgeig.cg import block_cg  # noqa: E402
from gcgeig.dense import sym_eig_full  # noqa: E402
from gcgeig.operators import CsrOperator, ShiftedOperator  # noqa: E402


def tridiag(n):
    return scipy.sparse.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1],
                              format="csr")


class patched:
    """BASELINE.md §3 patch of the reference: N(0,1) init + north-star residual."""

    def __enter__(self):
        self.saved = (S.mv_set_random, S._rel_residual)

        def normal(x, seed):
            x[...] = np.random.Generator(np.random.PCG64(seed)).standard_normal(x.shape)
            return x

        def rel(ax, x, bx, lam, generalized):
            r = ax - lam * bx
            den = abs(lam) * math.sqrt(float(bx @ bx))
            return math.sqrt(float(r @ r)) / (den if den != 0.0 else 1.0)

        S.mv_set_random, S._rel_residual = normal, rel
        return self

    def __exit__(self, *exc):
        S.mv_set_random, S._rel_residual = self.saved


def solver_cases():
    """(name, A, B, config kwargs, baseline_patch)."""
    fem_a, fem_b = P.fem_p1_cube(6)
    return [
        ("tri120", tridiag(120), None, dict(num_eigen=5, seed=13), False),
        ("lap2d20", P.laplacian_2d(20), None, dict(num_eigen=12, seed=1, tol=1e-9), False),
        ("fem6", fem_a, fem_b, dict(num_eigen=8, seed=2), False),
        ("tri200_moving", tridiag(200), None,
         dict(num_eigen=30, block_size=8, seed=7, moving=True), False),
        ("lap3d10_noshift", P.laplacian_3d(10), None,
         dict(num_eigen=20, seed=0, shift_mode="none"), False),
        ("lap3d12_baseline", P.laplacian_3d(12), None, dict(num_eigen=24, seed=0), True),
        ("fem8_baseline", *P.fem_p1_cube(8), dict(num_eigen=10, seed=0), True),
        ("varcoef10_moving", P.varcoef_diffusion_3d(10, seed=0), None,
         dict(num_eigen=40, seed=0, moving=True), True),
        ("cfg1_baseline", P.laplacian_2d(100), None,
         dict(num_eigen=20, block_size=20, tol=1e-8, seed=0), True),
    ]


def run_solver(a, b, kw, patch):
    if patch:
        with patched():
            return gcg_solve(a, b, SolverConfig(**kw))
    return gcg_solve(a, b, SolverConfig(**kw))


def small(out):
    rng = np.random.default_rng(0)
    # --- kernel KATs (test_kernels.py:25-102 shapes) under both backends
    m = scipy.sparse.random(120, 120, density=0.08, random_state=np.random.RandomState(2))
    m = (m + m.T).tocsr()
    m.sum_duplicates()
    out["k_csr_indptr"] = m.indptr.astype(np.int64)
    out["k_csr_indices"] = m.indices.astype(np.int64)
    out["k_csr_data"] = m.data
    out["k_csr_x"] = np.asfortranarray(rng.standard_normal((120, 7)))
    x5 = np.asfortranarray(np.random.default_rng(3).standard_normal((5000, 6)))
    y5 = np.asfortranarray(np.random.default_rng(31).standard_normal((5000, 4)))
    out["k_ip_x"], out["k_ip_y"] = x5, y5
    ax = np.asfortranarray(np.random.default_rng(5).standard_normal((200, 3)))
    ay = np.asfortranarray(np.random.default_rng(51).standard_normal((200, 3)))
    out["k_axpby_x"], out["k_axpby_y"] = ax, ay
    for be in K.available_backends():
        K.use_backend(be)
        o = np.zeros((120, 7), order="F")
        K.csr_matvec(out["k_csr_indptr"], out["k_csr_indices"], m.data, out["k_csr_x"], o)
        out[f"k_csr_out_{be}"] = o
        for det in (False, True):
            g = np.empty((6, 4), order="F")
            K.inner_product(x5, y5, g, 512, det)
            out[f"k_ip_out_{be}_{int(det)}"] = g.copy()
        for i, (al, bt) in enumerate([(0.0, 0.0), (1.0, 0.0), (0.0, 1.0), (2.5, 1.0), (2.5, -0.5)]):
            y = ay.copy(order="F")
            K.axpby(al, ax, bt, y)
            out[f"k_axpby_out_{be}_{i}"] = y
    K.use_backend("numpy")
    # --- block CG (test_cg.py shapes)
    op = CsrOperator(tridiag(60))
    rhs = np.asfortranarray(np.random.default_rng(2).uniform(-1, 1, (60, 4)))
    x0 = np.asfortranarray(np.random.default_rng(21).uniform(-1, 1, (60, 4)))
    w, rep = block_cg(ShiftedOperator(op, None, 0.05), rhs, x0=x0, max_iters=30, rel_tol=0.01)
    out["cg_rhs"], out["cg_x0"], out["cg_w"] = rhs, x0, w
    out["cg_meta"] = np.array([rep.iterations, rep.converged.sum(), rep.frozen.sum()])
    out["cg_relres"] = rep.relative_residuals
    # --- orth (test_orth.py: recursive counts 7 and 5, orth_against)
    for tag, seed, tol in (("strict", 303, 1e-15), ("default", 304, 1e-10)):
        xb = np.asfortranarray(np.random.default_rng(seed).uniform(-1, 1, (256, 32)))
        out[f"orth_{tag}_in"] = xb.copy(order="F")
        r = R.recursive_orth_svd(xb, cfg=R.OrthConfig(reorth_tol=tol))
        out[f"orth_{tag}_out"] = xb
        out[f"orth_{tag}_meta"] = np.array([r.num_kept, r.reduction_count])
    basis = np.asfortranarray(np.random.default_rng(51).uniform(-1, 1, (300, 40)))
    R.recursive_orth_svd(basis)
    xa = np.asfortranarray(np.random.default_rng(52).uniform(-1, 1, (300, 12)))
    xa[:, 5] = basis @ np.random.default_rng(53).uniform(-1, 1, 40)   # spanned column
    out["oa_basis"], out["oa_in"] = basis, xa.copy(order="F")
    r = R.orth_against(xa, basis)
    out["oa_out"], out["oa_meta"] = xa, np.array([r.num_kept, r.reduction_count])
    # --- dense (test_dense.py fixture_m8)
    raw = np.random.default_rng(2024).uniform(-1.0, 1.0, size=(8, 8))
    m8 = (raw + raw.T) / 2.0
    dec = sym_eig_full(m8)
    out["m8"], out["m8_values"], out["m8_vectors"] = m8, dec.values, dec.vectors
    # --- solver runs
    meta = {}
    for name, a, b, kw, patch in solver_cases():
        t0 = time.perf_counter()
        rep = run_solver(a, b, kw, patch)
        dt = time.perf_counter() - t0
        out[f"s_{name}_values"] = rep.eigenvalues
        out[f"s_{name}_residuals"] = rep.residuals
        if a.shape[0] <= 2000:
            out[f"s_{name}_vectors"] = rep.eigenvectors
        meta[name] = dict(
            kw=kw, baseline_patch=patch, status=rep.status, iterations=rep.iterations,
            total_reductions=rep.total_reductions, max_projection_dim=rep.max_projection_dim,
            converged=[h.num_converged for h in rep.history],
            cg=[h.cg_iterations for h in rep.history],
            theta=[h.theta for h in rep.history], seconds=dt,
        )
        print(f"{name}: {rep.status} iters={rep.iterations} {dt:.2f}s")
    return meta


def cfg_run(cfg):
    pr = P.baseline_problem(cfg)
    K.use_backend("numpy")
    t0 = time.perf_counter()
    with patched():
        rep = gcg_solve(pr.a, pr.b, SolverConfig(num_eigen=pr.num_eigen, block_size=pr.block_size,
                                                 tol=pr.tol, moving=pr.moving, seed=0))
    dt = time.perf_counter() - t0
    return dict(
        name=pr.name, status=rep.status, iterations=rep.iterations, seconds=dt,
        cpu_count=os.cpu_count(), backend="numpy",
        eigenvalues=rep.eigenvalues.tolist(), residuals=rep.residuals.tolist(),
        converged=[h.num_converged for h in rep.history],
        cg=[h.cg_iterations for h in rep.history],
        total_reductions=rep.total_reductions,
        step_seconds={k: sum(h.timings[k] for h in rep.history)
                      for k in rep.history[0].timings},
    )


def mid_cases():
    """Mid-size members of the config 4 / config 5 families (moving window), run by the
    reference with the BASELINE.md §3 patch: cfg4's variable-coefficient operator at 32^3
    (nev = 100) and cfg5's 27-point stencil at 64^3 (nev = 100, tol 1e-7) — the
    scaled-down cases the row-partitioned and arena tests compare against."""
    return [
        ("varcoef32_moving", P.varcoef_diffusion_3d(32, seed=0), None,
         dict(num_eigen=100, seed=0, moving=True, tol=1e-8)),
        ("stencil27_64_moving", P.stencil27(64), None,
         dict(num_eigen=100, seed=0, moving=True, tol=1e-7)),
    ]


def mid(names=None):
    K.use_backend("numpy")
    path = os.path.join(HERE, "golden_mid.json")
    res = json.load(open(path)) if os.path.exists(path) else {}
    for name, a, b, kw in mid_cases():
        if names and name not in names:
            continue
        t0 = time.perf_counter()
        rep = run_solver(a, b, kw, True)
        dt = time.perf_counter() - t0
        res[name] = dict(kw=kw, status=rep.status, iterations=rep.iterations, seconds=dt,
                         cpu_count=os.cpu_count(), backend="numpy",
                         eigenvalues=rep.eigenvalues.tolist(), residuals=rep.residuals.tolist(),
                         converged=[h.num_converged for h in rep.history],
                         total_reductions=rep.total_reductions,
                         max_projection_dim=rep.max_projection_dim)
        print(f"{name}: {rep.status} iters={rep.iterations} {dt:.1f}s", flush=True)
        with open(path, "w") as f:
            json.dump(res, f, indent=1)


def alg2_cases():
    """modified_block_orth (Alg. 2) inputs following test_orth.py:46-67, 145-178."""
    def blk(n, m, seed):
        return np.asfortranarray(np.random.default_rng(seed).uniform(-1.0, 1.0, (n, m)))
    cases = [
        ("m8_b2", blk(64, 8, 101), None, None, dict(block_width=2)),
        ("m32_b2", blk(256, 32, 202), None, None, dict(block_width=2)),
        ("m8_default", blk(64, 8, 103), None, None, {}),
    ]
    x = blk(40, 8, 21)
    x[:, 3] = x[:, 1]
    cases.append(("dup_col", x, None, None, dict(block_width=2)))
    x = blk(30, 6, 23)
    x[:, 4] = 0.0
    cases.append(("zero_col", x, None, None, dict(block_width=3)))
    cases.append(("with_b", blk(50, 8, 7), None, "tridiag50", {}))
    basis = blk(120, 10, 61)
    R.recursive_orth_svd(basis)
    cases.append(("with_x0", blk(120, 24, 62), basis, None, dict(block_width=5)))
    cases.append(("m96_b16", blk(600, 96, 63), None, None, dict(block_width=16)))
    return cases


def spd_tridiag(n):
    return scipy.sparse.diags([np.ones(n - 1), 4.0 * np.ones(n), np.ones(n - 1)], [-1, 0, 1],
                              format="csr")


def alg2(out):
    for tag, x, x0, bname, kw in alg2_cases():
        b = CsrOperator(spd_tridiag(50)) if bname == "tridiag50" else None
        out[f"{tag}_in"] = x.copy(order="F")
        if x0 is not None:
            out[f"{tag}_x0"] = x0
        r = R.modified_block_orth(x, x0=x0, b=b, cfg=R.OrthConfig(**kw))
        out[f"{tag}_out"] = x
        out[f"{tag}_meta"] = np.array([r.num_kept, r.reduction_count])
        out[f"{tag}_replaced"] = np.array(r.replaced_indices, dtype=np.int64)
        print(f"alg2 {tag}: kept={r.num_kept} reductions={r.reduction_count}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=0, help="full BASELINE config run (2 or 3)")
    ap.add_argument("--alg2", action="store_true", help="only the Alg. 2 vectors -> golden_alg2.npz")
    ap.add_argument("--mid", nargs="*", default=None,
                    help="mid-size cfg4/cfg5-family moving-window runs -> golden_mid.json")
    args = ap.parse_args()
    if args.mid is not None:
        mid(args.mid)
        return
    if args.alg2 or not args.cfg:
        o2 = {}
        alg2(o2)
        np.savez_compressed(os.path.join(HERE, "golden_alg2.npz"), **o2)
        if args.alg2:
            return
    if args.cfg:
        res = cfg_run(args.cfg)
        with open(os.path.join(HERE, f"golden_cfg{args.cfg}.json"), "w") as f:
            json.dump(res, f, indent=1)
        print(f"cfg{args.cfg}", res["status"], res["iterations"], f"{res['seconds']:.1f}s")
        return
    out = {}
    meta = small(out)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(dict(generator="tests/golden/make_golden.py", reference="gcgeig " + gcgeig.__version__,
                       numpy=np.__version__, scipy=scipy.__version__, solver=meta), f, indent=1)


if __name__ == "__main__":
    main()
