"""GCG iteration counts of the golden solver cases on the B200 vs the reference's (development helper)."""
import json, os, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2111_06552_b200 import SolverConfig, gcg_solve
from tests.cases import SOLVER_CASES, problem
meta = json.load(open("tests/golden/golden.json"))["solver"]
for name in SOLVER_CASES:
    m = meta[name]
    a, b = problem(name)
    kw = dict(m["kw"])
    if m["baseline_patch"]:
        kw.update(init="normal", residual="relative")
    rep = gcg_solve(a, b, SolverConfig(**kw))
    print(f"{name:32s} gpu {rep.iterations:4d}  reference {m['iterations']:4d}")
