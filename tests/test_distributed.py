"""Row-partition bookkeeping and the collectives of the multi-GPU path, on CPU.

* local_part: every rank's local CSR applied to [owned rows | ghost rows] of a
  vector equals the corresponding rows of the global product, and the halo
  lists are consistent (what p sends to q is exactly what q expects from p);
* Comm over gloo with world_size 2 (two processes on 127.0.0.1): point-to-point
  exchange, ordered all-gather sum (identical on both ranks), broadcast.
"""

import os
import socket

import numpy as np
import pytest
import scipy.sparse
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2111_06552_b200 import problems as P
from paper_2111_06552_b200.distributed import Comm, local_part, row_bounds


def _global_rows(part):
    return np.concatenate([np.arange(part.r0, part.r0 + part.nloc), part.ghost_global])


@pytest.mark.parametrize("nranks", [1, 2, 3, 4])
@pytest.mark.parametrize("which", ["lap3d", "fem", "rand"])
def test_local_part_reproduces_global_rows(nranks, which):
    b = None
    if which == "lap3d":
        a = P.laplacian_3d(9)
        plane = 81
    elif which == "fem":
        a, b = P.fem_p1_cube(6)
        plane = 25
    else:
        m = scipy.sparse.random(150, 150, density=0.04, random_state=np.random.RandomState(3))
        a = (m + m.T + scipy.sparse.eye(150)).tocsr()
        plane = 1
    n = a.shape[0]
    bounds = row_bounds(n, nranks, plane)
    assert bounds[0] == 0 and bounds[-1] == n and np.all(np.diff(bounds) > 0)
    x = np.random.default_rng(0).standard_normal((n, 3))
    ya = a @ x
    parts = [local_part(a, b, bounds, r) for r in range(nranks)]
    for part in parts:
        xl = x[_global_rows(part)]
        assert np.allclose(part.a @ xl, ya[part.r0:part.r0 + part.nloc], rtol=0, atol=1e-12)
        if b is not None:
            yb = b @ x
            assert np.allclose(part.b @ xl, yb[part.r0:part.r0 + part.nloc], rtol=0, atol=1e-14)
            assert np.array_equal(part.a.indices, part.b.indices)
    # halo consistency: p sends to q exactly the ghost rows q expects from p, in order
    for p in parts:
        for q in parts:
            if p.rank == q.rank:
                continue
            sent = p.send_rows[q.rank] + p.r0
            lo = int(np.sum(q.recv_counts[:p.rank]))
            expect = q.ghost_global[lo:lo + q.recv_counts[p.rank]]
            assert np.array_equal(sent, expect)


def test_row_bounds_plane_alignment():
    b = row_bounds(64 ** 3, 8, 64 * 64)
    assert np.all(b % (64 * 64) == 0)
    b = row_bounds(10, 3)
    assert list(b) == [0, 3, 6, 10]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = Comm()
        # point to point: each rank sends (rank+1)*[1..4] to the other
        other = 1 - rank
        sends = [None, None]
        recvs = [None, None]
        sends[other] = torch.arange(1, 5, dtype=torch.float64) * (rank + 1)
        recvs[other] = torch.zeros(4, dtype=torch.float64)
        comm.exchange(sends, recvs)
        got = recvs[other].tolist()
        # ordered sum: values chosen so a different order would round differently
        t = torch.tensor([1e16, 1.0, -1e16], dtype=torch.float64) if rank == 0 else \
            torch.tensor([1.0, 1e16, 1.0], dtype=torch.float64)
        comm.allgather_sum(None, t)
        s = t.tolist()
        bt = torch.tensor([float(rank + 7)], dtype=torch.float64)
        comm.broadcast(bt, src=1)
        # allreduce mode (the paper's SUBMAT allreduce): same result on both ranks
        ar = Comm(reduce="allreduce")
        u = torch.tensor([0.5, 2.0, -3.0], dtype=torch.float64) * (rank + 1)
        ar.allgather_sum(None, u)
        q.put((rank, got, s, bt.item(), u.tolist()))
    finally:
        dist.destroy_process_group()


def test_comm_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(2):
        r, got, s, b, u = q.get(timeout=120)
        res[r] = (got, s, b, u)
    for p in procs:
        p.join(timeout=60)
    assert res[0][0] == [2.0, 4.0, 6.0, 8.0]
    assert res[1][0] == [1.0, 2.0, 3.0, 4.0]
    assert res[0][1] == res[1][1]                     # bit-identical on both ranks
    assert res[0][1] == [1e16 + 1.0, 1.0 + 1e16, -1e16 + 1.0]
    assert res[0][2] == res[1][2] == 8.0
    assert res[0][3] == res[1][3] == [1.5, 6.0, -9.0]


def test_cfg5_memory_plan_fits_at_4_and_8_gpus():
    """BASELINE config 5 (27-pt 256^3, nev = 1000, moving): the per-rank HBM plan of the
    single-arena solver fits a 180 GB B200 with headroom at 4 and 8 ranks
    and does not at 1 or 2 — the SURVEY §8(d) memory analysis."""
    from paper_2111_06552_b200.solver import device_memory_plan

    n, nnz, plane = 256 ** 3, 449_455_096, 256 * 256
    gb = {}
    for ranks in (1, 2, 4, 8):
        nloc = n // ranks
        nghost = 0 if ranks == 1 else 2 * plane
        plan = device_memory_plan(nloc, nnz // ranks + 1, 1000, moving=True, nghost=nghost)
        gb[ranks] = plan["total"] / 1e9
    assert gb[4] < 170.0 and gb[8] < 90.0
    assert gb[2] > 180.0 and gb[1] > 180.0
