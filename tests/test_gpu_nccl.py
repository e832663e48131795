"""The library's own NCCL communicator (csrc/nccl.cu) on the GPU box.

Only one GPU is available to the tests and NCCL refuses two ranks on one device, so
this runs the row-partitioned solver as a one-rank NCCL job: the communicator is
bootstrapped through the torch process group, and every block-CG sweep's halo and
k-vector sums go through gcg_nccl_* on the library stream (no Python callback) —
the data path of a multi-GPU run, minus the peers.  The result must match the
reference golden run like the single-GPU solve does."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_2111_06552_b200 import SolverConfig, _lib
        from paper_2111_06552_b200 import device as D
        from paper_2111_06552_b200.distributed import Comm, gcg_solve_distributed
        from tests.cases import problem

        ver = int(_lib.load().gcg_nccl_available())
        comm = Comm()
        native = comm.native is not None
        # the raw collective on the library stream
        dev = D.default_context()
        t = torch.arange(7, dtype=torch.float64, device=dev.device)
        comm.native.allreduce_sum(t)
        torch.cuda.synchronize()
        same = bool(torch.equal(t.cpu(), torch.arange(7, dtype=torch.float64)))
        a, b = problem("lap3d12_baseline")
        kw = dict(num_eigen=24, seed=0, init="normal", residual="relative")
        rep = gcg_solve_distributed(a, b, SolverConfig(**kw), comm=comm, plane=144)
        comm.close()
        q.put(("ok", ver, native, same, rep.status, rep.iterations, rep.eigenvalues,
               rep.residuals))
    except Exception as exc:  # report instead of hanging the parent
        q.put(("error", repr(exc)))
    finally:
        dist.destroy_process_group()


def test_native_nccl_single_rank_solve(golden, golden_meta):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(_free_port(), q))
    p.start()
    res = q.get(timeout=600)
    p.join(timeout=120)
    assert res[0] == "ok", res
    _, ver, native, same, status, iters, vals, resid = res
    assert ver > 0 and native and same
    assert status == "converged"
    want = golden["s_lap3d12_baseline_values"]
    assert np.abs(vals - want).max() <= 1e-9 * max(1.0, np.abs(want).max())
    assert resid.max() < 1e-8
    meta = golden_meta["solver"]["lap3d12_baseline"]
    assert abs(iters - meta["iterations"]) <= max(4, int(0.15 * meta["iterations"]))
