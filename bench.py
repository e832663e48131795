"""Benchmark: time-to-nev of the GCG eigensolver on the B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl reference]

A step is one complete solve (time-to-nev) of BASELINE config 2 — the 3-D
7-point Laplacian on 64^3 (n = 262,144), nev = 100, tol 1e-8, N(0,1) initial
block from seed 0, north-star residual criterion — through the drop-in
`gcg_solve`.  `value` is the device-timed solve with the matrix and the seeded
initial block already resident in HBM; `e2e` times the public call with host
buffers (CSR + initial block H2D, eigenpairs D2H inside the timed region).

--impl reference times the reference's own CPU implementation (the unmodified
gcgeig built into oracle/_ref by oracle/build_ref.sh, else the oracle port) on
a bounded sample (a few GCG iterations per step) and extrapolates to the
reference's full iteration count; see DESIGN.md §6.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-to-nev (s)"
UNIT = "s"


PROF_SAMPLE = 4  # time every 4th launch of each kernel class (see KernelProfile)
REF_BUDGET_S = 150.0  # CPU seconds the reference arm may spend on timed samples


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def solver_kwargs(pr):
    return dict(num_eigen=pr.num_eigen, block_size=pr.block_size, tol=pr.tol, moving=pr.moving,
                seed=0)


def problem_size(pr):
    """(n, nnz(A)) — from the matrix, or from the generator for device-assembled configs."""
    if pr.a is not None:
        return pr.a.shape[0], int(pr.a.nnz)
    from paper_2111_06552_b200 import _lib
    import ctypes as C
    import itertools

    N = pr.grid[0]
    offs = list(itertools.product((-1, 0, 1), repeat=3))
    flat = (C.c_int32 * (3 * len(offs)))(*[v for o in offs for v in o])
    nnz = C.c_int64()
    _lib.call("gcg_stencil_nnz", N, N, N, len(offs), flat, C.byref(nnz))
    return N ** 3, int(nnz.value)


def bench_config(pr, world):
    """The `config` dict both arms print (identical keys, so the driver's same_config holds)."""
    n, nnz = problem_size(pr)
    return {"workload": pr.name, "n": n, "nnz": nnz,
            "nev": pr.num_eigen, "tol": pr.tol, "criterion": "north-star relative",
            "parallelism": f"row-partition x{world} (z-slabs, halo + reductions)"
            if world > 1 else "single",
            "l2": "working set (arena + CG blocks) > 126 MB L2, no flush"}


def initial_block(pr):
    """The seeded N(0,1) block both arms start from."""
    n = pr.a.shape[0]
    bs = pr.block_size or max(1, -(-pr.num_eigen // 5))
    sx = min(3 * bs, n) if pr.moving else min(pr.num_eigen + 3 * bs, n)
    return np.random.Generator(np.random.PCG64(0)).standard_normal((n, sx))


# ---------------------------------------------------------------------------
# clocks sampled during the timed region


class ClockSampler:
    REASONS = {
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
        0x2: "applications_clocks_setting", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.index = index
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons)}


# ---------------------------------------------------------------------------
# CPU reference arm


def reference_solver():
    """(gcg_solve, SolverConfig, kind) of the reference, patched per BASELINE.md §3."""
    import oracle

    g = oracle.load_reference()
    if g is not None:
        import math

        from gcgeig import SolverConfig, gcg_solve
        from gcgeig import _kernels as K
        from gcgeig import solver as S

        def normal(x, seed):
            x[...] = np.random.Generator(np.random.PCG64(seed)).standard_normal(x.shape)
            return x

        def rel(ax, x, bx, lam, generalized):
            r = ax - lam * bx
            den = abs(lam) * math.sqrt(float(bx @ bx))
            return math.sqrt(float(r @ r)) / (den if den != 0.0 else 1.0)

        S.mv_set_random, S._rel_residual = normal, rel
        K.use_backend("numpy")  # multithreaded BLAS beats the 1-thread Cython core at scale

        def run(a, b, kw):
            return gcg_solve(a, b, SolverConfig(**kw))

        return run, "reference"
    from oracle import gcg_oracle as O

    def run(a, b, kw):
        return O.gcg_solve(a, b, O.OracleConfig(**kw, init="normal", residual="relative"))

    return run, "port"


def reference_iterations(cfg):
    """Full-solve GCG iteration count of the reference (committed golden run), if known."""
    path = os.path.join(ROOT, "tests", "golden", f"golden_cfg{cfg}.json")
    if os.path.exists(path):
        return int(json.load(open(path))["iterations"]), "reference full solve (tests/golden)"
    return None, None


def cpu_sample(pr, iters, cfg):
    """Time `iters` GCG iterations of the reference on this host; extrapolate time-to-nev."""
    run, kind = reference_solver()
    kw = solver_kwargs(pr)
    kw["max_gcg_iters"] = iters
    t0 = time.perf_counter()
    run(pr.a, pr.b, kw)
    dt = time.perf_counter() - t0
    full, src = reference_iterations(cfg)
    return dt, kind, full, src


def run_reference_arm(args, pr, rank, world):
    """Each step times the reference for 1 and for 2 GCG iterations: the difference is one
    iteration, the rest its setup (initial draw + orthogonalisation), counted once:
    time-to-nev = t(1) + (full - 1) * (t(2) - t(1))."""
    if rank != 0:
        return
    # bounded: one untimed 1-iteration warm-up, then (1-iteration, 2-iteration) sample pairs
    # until K pairs or REF_BUDGET_S seconds of CPU time, at least one pair
    t1s, t2s = [], []
    kind = full = src = None
    if args.warmup > 0:
        cpu_sample(pr, 1, args.config)
    t_start = time.perf_counter()
    for s in range(max(1, args.steps)):
        dt1, kind, full, src = cpu_sample(pr, 1, args.config)
        dt2, kind, full, src = cpu_sample(pr, 2, args.config)
        t1s.append(dt1)
        t2s.append(dt2)
        if time.perf_counter() - t_start > REF_BUDGET_S:
            break
    t1, t2 = statistics.mean(t1s), statistics.mean(t2s)
    per_iter = max(t2 - t1, 1e-9)
    if full is None:
        full = 43
        src = "assumed 43 iterations"
    value = t1 + (full - 1) * per_iter
    times = [a + b for a, b in zip(t1s, t2s)]
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * value,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE generator, seeded N(0,1) initial block)",
        "config": bench_config(pr, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{len(t1s)} pair(s) of 1- and 2-iteration runs (setup "
                                   f"{t1 - per_iter:.2f} s + {per_iter:.2f} s/iter), extrapolated "
                                   f"to {full} iterations ({src})"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gcg_iters_per_s": 1.0 / per_iter,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm


def main():
    args = parse()
    rank, world, local = dist_env()
    from paper_2111_06552_b200 import problems as P

    # config 5 (449 M nonzeros, nev = 1000) is only ever assembled on the devices, one
    # z-slab per rank; it needs >= 4 GPUs (device_memory_plan)
    device_built = args.config == 5
    pr = P.baseline_problem(args.config, build=not device_built)
    if args.impl == "reference":
        if device_built:
            if rank == 0:
                print(json.dumps({"impl": "reference", "unavailable":
                                  "config 5 needs > 300 GB of host memory for the reference "
                                  "(SURVEY §8(d)); not runnable on this host"}), flush=True)
            return
        run_reference_arm(args, pr, rank, world)
        return

    import torch
    import torch.distributed as dist

    # one GPU per rank; GCG_BENCH_BACKEND=gloo lets several ranks share a GPU (testing only)
    backend = os.environ.get("GCG_BENCH_BACKEND", "nccl")
    dev_index = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev_index)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
    from paper_2111_06552_b200 import SolverConfig, _lib, gcg_solve
    from paper_2111_06552_b200 import device as D
    from paper_2111_06552_b200.operators import as_device_problem
    from paper_2111_06552_b200.solver import gcg_solve_ops

    ctx = D.default_context()
    kw = solver_kwargs(pr)
    n_glob, nnz_glob = problem_size(pr)
    if device_built:
        from paper_2111_06552_b200.solver import device_memory_plan

        plane = pr.grid[1] * pr.grid[2]
        plan = device_memory_plan(n_glob // world, nnz_glob // world + 1, pr.num_eigen,
                                  moving=pr.moving, nghost=0 if world == 1 else 2 * plane)
        cap = torch.cuda.get_device_properties(dev_index).total_memory
        if plan["total"] > 0.95 * cap:
            if rank == 0:
                print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world,
                                  "config": bench_config(pr, world), "unavailable":
                                  f"per-rank HBM plan {plan['total'] / 1e9:.0f} GB > device "
                                  f"{cap / 1e9:.0f} GB at {world} GPU(s); config 5 runs at >= 4"}),
                      flush=True)
            if world > 1:
                dist.destroy_process_group()
            return
    # the seeded N(0,1) initial block: host PCG64 (the reference's stream) where a host
    # draw is affordable, the partition-invariant device draw for config 5
    x0_host = None if device_built else initial_block(pr)
    cfg = SolverConfig(**kw, init="philox" if device_built else "normal", residual="relative",
                       validate=False, return_device=True, collect_history=True)
    plane = int(np.prod(pr.grid[1:])) if len(pr.grid) > 1 else 1
    if world > 1:
        # row-partitioned solve: z-slab row blocks, halo exchange + NCCL reductions; the
        # structured-grid operators are assembled per rank on the device (no global host CSR)
        from paper_2111_06552_b200.distributed import (Comm, DistOps, DistProblem, local_part,
                                                       row_bounds, slab_problem)

        comm = Comm()
        if args.config in (1, 2, 4, 5):
            dprob, _ = slab_problem(ctx, comm, args.config)
        else:
            bounds = row_bounds(n_glob, world, plane)
            dprob = DistProblem(ctx, local_part(pr.a, pr.b, bounds, rank), comm, n_glob)
        ops = DistOps(ctx, dprob)
        x0_local = None if x0_host is None else x0_host[ops.row0:ops.row0 + ops.nloc]
    else:
        from paper_2111_06552_b200.mvops import LocalOps

        if device_built:
            from paper_2111_06552_b200.devgen import device_baseline_problem

            ops = LocalOps(ctx, device_baseline_problem(ctx, args.config)[0])
        else:
            ops = LocalOps(ctx, as_device_problem(ctx, pr.a, pr.b, validate=False))
        x0_local = x0_host
    x0_dev = None if x0_local is None else \
        torch.from_numpy(np.ascontiguousarray(x0_local)).to(ctx.device)

    def step():
        return gcg_solve_ops(ops, cfg, x0=x0_dev)

    for _ in range(args.warmup):
        rep = step()
    barrier = (lambda: dist.barrier()) if world > 1 else (lambda: None)
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.launch_count()
    iters = []
    # per-kernel CUDA events on every 4th launch of each class: the roofline is measured
    # live inside the timed region while perturbing it ~4x less than timing every launch
    with ClockSampler(dev_index) as clk, D.KernelProfile(ctx, sample=PROF_SAMPLE) as prof:
        ev0.record(ctx.stream)
        for _ in range(args.steps):
            rep = step()
            iters.append(rep.iterations)
        ev1.record(ctx.stream)
        torch.cuda.synchronize()
    barrier()
    launches = _lib.launch_count() - l0
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=ctx.device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    t_solve = ms / 1e3 / args.steps
    assert rep.status == "converged" and rep.residuals.max() <= pr.tol, (rep.status, rep.residuals.max())

    # end-to-end through the public call with host buffers (pinned CSR + x0 in, eigenpairs out)
    e2e = None
    if not args.no_e2e and not device_built:
        import scipy.sparse

        # inputs in pinned host memory: the CSR arrays (int32 indices, as the device stores
        # them) are numpy views of page-locked torch buffers, so the upload is a DMA
        def pinned(arr):
            t = torch.empty(arr.shape, dtype=torch.from_numpy(arr[:0]).dtype, pin_memory=True)
            out = t.numpy()
            out[...] = arr
            return out

        src = scipy.sparse.csr_matrix(pr.a)
        a_pinned = scipy.sparse.csr_matrix(
            (pinned(src.data.astype(np.float64)), pinned(src.indices.astype(np.int32)),
             pinned(src.indptr.astype(np.int32))), shape=src.shape)
        x0_pin = torch.from_numpy(np.ascontiguousarray(x0_local)).pin_memory()
        # validate=True: the symmetry / finiteness check the reference runs inside its
        # operator construction (operators.py:79-96) stays inside the timed call
        cfg_h = SolverConfig(**kw, init="normal", residual="relative", validate=True)
        rows = slice(ops.row0, ops.row0 + ops.nloc)
        nnz_local = int(a_pinned.indptr[rows.stop] - a_pinned.indptr[rows.start])
        h2d = 12 * nnz_local + 4 * (ops.nloc + 1) + x0_pin.numel() * 8
        if pr.b is not None:
            h2d += 8 * nnz_local
        torch.cuda.synchronize()
        barrier()
        te = []
        # W untimed warm-up calls (first-call host costs: pinned staging, page faults),
        # then K timed calls, as for the device-timed value
        for i in range(args.warmup + max(1, args.steps)):
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            if world > 1:
                from paper_2111_06552_b200.distributed import gcg_solve_distributed

                rh = gcg_solve_distributed(a_pinned, pr.b, cfg_h, comm=comm, plane=plane,
                                           x0=x0_pin)
            else:
                rh = gcg_solve(a_pinned, pr.b, cfg_h, x0=x0_pin)
            torch.cuda.synchronize()
            if i >= args.warmup:
                te.append(time.perf_counter() - t0)
        if os.environ.get("GCG_BENCH_DEBUG"):
            print("e2e steps (s):", [round(v, 4) for v in te], file=sys.stderr)
        d2h = rh.eigenvectors.nbytes + rh.eigenvalues.nbytes + rh.residuals.nbytes
        e_val = statistics.mean(te)
        if world > 1:
            t = torch.tensor([e_val], device=ctx.device, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_val = float(t.item())
        e2e = {"value": e_val, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h)}

    # roofline of the dominant kernel class (live CUDA-event timing inside the timed region)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    res = prof.result
    dom = max(res, key=lambda k: res[k]["ms"])
    r = res[dom]
    achieved = (r["bytes"] / r["launches"]) / (r["ms"] / r["launches"] / 1e3) / 1e9 if r["launches"] else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(dom)
    kernels = {k: {"ms_per_step": v["ms"] * PROF_SAMPLE / args.steps,
                   "launches_per_step": v["launches"] * PROF_SAMPLE / args.steps,
                   "GBps": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 else 0.0}
               for k, v in res.items()}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            dt1, kind, full, src = cpu_sample(pr, 1, args.config)
            dt2, kind, full, src = cpu_sample(pr, 2, args.config)
            per_iter = max(dt2 - dt1, 1e-9)
            if full is None:
                full, src = rep.iterations, "this run's GPU iteration count"
            cpu = {"value": dt1 + (full - 1) * per_iter, "unit": UNIT, "cores": os.cpu_count(),
                   "kind": kind,
                   "sample": f"1- and 2-iteration runs of {pr.name} ({dt1:.1f} s, {dt2:.1f} s; "
                             f"{'gcgeig numpy backend' if kind == 'reference' else 'oracle port'}): "
                             f"setup {dt1 - per_iter:.1f} s + {per_iter:.2f} s/iter, extrapolated "
                             f"to {full} iterations ({src}); the GPU value excludes drawing the "
                             f"initial block, the reference's setup includes it"}
        except Exception as exc:  # keep the GPU line even if the CPU leg fails
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {exc!r}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": t_solve, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE generator, seeded N(0,1) initial block)",
            "config": bench_config(pr, world),
            "iterations": iters[-1], "gcg_iters_per_s": iters[-1] / t_solve,
            "max_residual": float(rep.residuals.max()),
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback",
                         "timing": f"CUDA events on every {PROF_SAMPLE}th launch of the class, "
                                   "inside the timed region"},
            "kernels": kernels,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
