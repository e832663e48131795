"""One measured full solve of the unmodified reference (oracle/_ref, patched per
BASELINE.md §3: N(0,1) initial block, north-star residual) on this host, all cores
(numpy backend, multithreaded BLAS) — the un-extrapolated CPU time-to-nev that
bench.py's 1/2-iteration samples extrapolate to.  Usage: ref_full_solve.py [cfg]."""
import json
import os
import platform
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2111_06552_b200 import problems as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pr = P.baseline_problem(cfg)
run, kind = bench.reference_solver()
kw = bench.solver_kwargs(pr)
t0 = time.perf_counter()
rep = run(pr.a, pr.b, kw)
dt = time.perf_counter() - t0
cpu = "unknown"
try:
    for line in open("/proc/cpuinfo"):
        if line.startswith("model name"):
            cpu = line.split(":", 1)[1].strip()
            break
except OSError:
    pass
out = {"config": cfg, "kind": kind, "seconds": dt, "iterations": int(rep.iterations),
       "status": rep.status, "cores": os.cpu_count(), "cpu": cpu, "host": platform.node(),
       "max_residual": float(np.max(rep.residuals))}
gold = os.path.join(bench.ROOT, "tests", "golden", f"golden_cfg{cfg}.json")
if os.path.exists(gold):
    want = np.array(json.load(open(gold))["eigenvalues"])
    out["max_rel_eig_diff_vs_golden"] = float(np.abs(rep.eigenvalues - want).max() / np.abs(want).max())
print(json.dumps(out), flush=True)
