"""Row-partitioned multi-GPU GCG: one process per GPU.

Partition: contiguous row blocks of A, B and every multivector (for the
BASELINE grids — rows in lexicographic order, first axis slowest — these are
z-slabs, so the halo of the 5/7/15/27-point operators is one grid plane per
side).  The small projected matrices are replicated.

Communication goes through torch.distributed:

* halo exchange before every SpMM: each rank packs the owned rows its
  neighbours reference (gcg_gather_rows), exchanges them point to point and
  writes them into the ghost rows that follow its local rows;
* Gram blocks / column sums: all-gather of the k1 x k2 partials and an ordered
  sum on device — identical bits on every rank (so every replica takes the same
  host-side decisions) and deterministic run to run;
* the Rayleigh-Ritz eigenvectors are broadcast from rank 0.

With NCCL (one GPU per rank, NVLink/NVSwitch) the collectives read and write
device memory directly; with gloo (CPU tests, or several ranks sharing one GPU)
device tensors are staged through host memory.
"""

from __future__ import annotations

import os

import ctypes as C
from dataclasses import dataclass

import numpy as np
import scipy.sparse
import torch
import torch.distributed as dist

from . import _lib
from . import device as D
from .mvops import LocalOps
from .operators import DeviceCsr, DeviceProblem, _shared_pattern

__all__ = ["row_bounds", "LocalPart", "local_part", "SlabPart", "slab_problem", "Comm",
           "DistProblem", "DistOps", "gcg_solve_distributed"]


def row_bounds(n, nranks, plane=1):
    """Balanced contiguous row blocks, aligned to multiples of `plane` rows when possible."""
    units = n // plane if plane > 1 and n % plane == 0 else n
    unit = plane if units != n else 1
    cuts = [(units * r) // nranks * unit for r in range(nranks + 1)]
    cuts[-1] = n
    return np.asarray(cuts, dtype=np.int64)


@dataclass
class LocalPart:
    """Host-side description of one rank's rows (pure index bookkeeping)."""

    rank: int
    bounds: np.ndarray           # row cut points, len = nranks + 1
    a: scipy.sparse.csr_matrix   # local rows, columns remapped: owned 0..nloc-1, ghosts after
    b: scipy.sparse.csr_matrix | None
    ghost_global: np.ndarray     # global row ids of the ghost rows (sorted)
    recv_counts: np.ndarray      # ghosts received from each rank
    send_rows: list              # per rank: local row ids to send (sorted)

    @property
    def r0(self):
        return int(self.bounds[self.rank])

    @property
    def nloc(self):
        return int(self.bounds[self.rank + 1] - self.bounds[self.rank])

    @property
    def nghost(self):
        return int(self.ghost_global.shape[0])


def local_part(a, b, bounds, rank):
    """Slice rows of A (and B on A's pattern) for `rank`, remap columns, build the halo lists.

    Requires a symmetric sparsity pattern (true for every operator here): the rows
    rank q needs from me are then exactly my rows that reference q's rows.
    """
    a = scipy.sparse.csr_matrix(a)
    if b is not None:
        a, b = _shared_pattern(a, b)
    nranks = len(bounds) - 1
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    nloc = r1 - r0
    sub = a[r0:r1].tocsr()
    sub.sort_indices()
    cols = sub.indices.astype(np.int64)
    outside = (cols < r0) | (cols >= r1)
    ghost = np.unique(cols[outside])
    newcols = np.where(outside, nloc + np.searchsorted(ghost, cols), cols - r0)
    owner_g = np.searchsorted(bounds, ghost, side="right") - 1
    recv_counts = np.bincount(owner_g, minlength=nranks).astype(np.int64)
    rows_of_nz = np.repeat(np.arange(nloc, dtype=np.int64), np.diff(sub.indptr))
    owner_nz = np.searchsorted(bounds, cols, side="right") - 1
    send_rows = []
    for q in range(nranks):
        if q == rank:
            send_rows.append(np.zeros(0, dtype=np.int64))
            continue
        send_rows.append(np.unique(rows_of_nz[owner_nz == q]))
    la = scipy.sparse.csr_matrix((sub.data, newcols.astype(np.int32), sub.indptr),
                                 shape=(nloc, nloc + ghost.shape[0]))
    lb = None
    if b is not None:
        bsub = b[r0:r1].tocsr()
        bsub.sort_indices()
        lb = scipy.sparse.csr_matrix((bsub.data, newcols.astype(np.int32), bsub.indptr),
                                     shape=la.shape)
    return LocalPart(rank, np.asarray(bounds), la, lb, ghost, recv_counts, send_rows)


@dataclass
class SlabPart:
    """LocalPart of a z-slab assembled on the device (devgen.stencil_slab_device): the same
    halo bookkeeping without host matrices — ghosts are the plane below (from rank - 1)
    and the plane above (from rank + 1); the rows sent are the slab's first / last plane."""

    rank: int
    bounds: np.ndarray
    nprev: int
    nnext: int
    a = None
    b = None

    @property
    def r0(self):
        return int(self.bounds[self.rank])

    @property
    def nloc(self):
        return int(self.bounds[self.rank + 1] - self.bounds[self.rank])

    @property
    def nghost(self):
        return self.nprev + self.nnext

    @property
    def recv_counts(self):
        c = np.zeros(len(self.bounds) - 1, dtype=np.int64)
        if self.nprev:
            c[self.rank - 1] = self.nprev
        if self.nnext:
            c[self.rank + 1] = self.nnext
        return c

    @property
    def send_rows(self):
        out = [np.zeros(0, dtype=np.int64) for _ in range(len(self.bounds) - 1)]
        if self.nprev:   # my first plane is the lower neighbour's upper ghost plane
            out[self.rank - 1] = np.arange(self.nprev, dtype=np.int64)
        if self.nnext:   # my last plane is the upper neighbour's lower ghost plane
            out[self.rank + 1] = np.arange(self.nloc - self.nnext, self.nloc, dtype=np.int64)
        return out


def slab_problem(dev, comm, cfg, scale=None, plane_align=True):
    """This rank's DistProblem of BASELINE config 1/2/4/5 assembled on the device: the
    global operator is never built on any host (config 5: 449 M nonzeros)."""
    from .devgen import baseline_stencil_spec, stencil_slab_device

    shape, offs, weights, meta = baseline_stencil_spec(dev, cfg, scale)
    n = int(np.prod(shape))
    plane = int(np.prod(shape[1:])) if plane_align else 1
    bounds = row_bounds(n, comm.size, plane)
    r0, r1 = int(bounds[comm.rank]), int(bounds[comm.rank + 1])
    A, nprev, nnext = stencil_slab_device(dev, shape, offs, weights, r0, r1)
    part = SlabPart(comm.rank, bounds, nprev, nnext)
    return DistProblem(dev, part, comm, n, A=A), meta


class NativeNccl:
    """One ncclComm_t created inside libgcgb200 (gcg_nccl_comm_create), bootstrapped by
    broadcasting rank 0's unique id over the torch process group."""

    def __init__(self, comm):
        dev = D.default_context()
        if not _lib.load().gcg_nccl_available():
            raise _lib.DeviceError("libnccl.so.2 could not be loaded for the native communicator")
        uid = (C.c_uint8 * 128)()
        if comm.rank == 0:
            _lib.call("gcg_nccl_unique_id", uid)
        t = torch.tensor(list(uid), dtype=torch.uint8, device=dev.device)
        dist.broadcast(t, src=0, group=comm.group)
        uid = (C.c_uint8 * 128)(*t.cpu().tolist())
        h = C.c_void_p()
        _lib.call("gcg_nccl_comm_create", dev.h, comm.size, comm.rank, uid, C.byref(h))
        self.handle = h
        self.dev = dev

    def allreduce_sum(self, t):
        """In-place sum of a contiguous float64 device tensor, on the library stream."""
        _lib.call("gcg_nccl_allreduce_sum", self.dev.h, self.handle, C.c_void_p(t.data_ptr()),
                  t.numel())
        return t

    def close(self):
        if self.handle:
            _lib.load().gcg_nccl_comm_destroy(self.handle)
            self.handle = None


class Comm:
    """Collectives over a torch.distributed process group.

    reduce="allgather" (default on host-staged backends): sums are all-gathered and
    added in rank order on every rank — bit-identical on all ranks and independent of
    the collective algorithm (the reference's deterministic mode, multivec.py:84-112).
    reduce="allreduce" (default with NCCL): one NCCL allreduce (the paper's SUBMAT
    allreduce) — every rank receives the same reduced bits, 1/P of
    the all-gather's bytes.  GCG_DIST_REDUCE overrides.
    """

    def __init__(self, group=None, reduce=None, native=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        self.staged = self.backend != "nccl"
        # NCCL: one allreduce (the paper's SUBMAT allreduce; every rank receives the same
        # reduced bits); host-staged backends: the all-gather + rank-ordered sum
        self.reduce = reduce or os.environ.get(
            "GCG_DIST_REDUCE", "allreduce" if self.backend == "nccl" else "allgather")
        if self.reduce not in ("allgather", "allreduce"):
            raise ValueError(f"unknown reduce mode {self.reduce!r}")
        # the library's own NCCL communicator (nccl.cu) for the block-CG halo and
        # reductions, so a distributed CG runs without host callbacks; on by default
        # with the NCCL backend (GCG_NATIVE_NCCL=0 keeps the Python callbacks)
        if native is None:
            native = self.backend == "nccl" and os.environ.get("GCG_NATIVE_NCCL", "1") != "0"
        self.native = None
        if native:
            self.native = NativeNccl(self)

    def close(self):
        if self.native is not None:
            self.native.close()
            self.native = None

    def _host(self, t):
        return t.cpu() if (self.staged and t.is_cuda) else t

    def allgather_sum(self, dev, t):
        """Sum of `t` over ranks, accumulated in rank order (identical bits everywhere);
        one allreduce instead in reduce="allreduce" mode."""
        if self.size == 1:
            return t
        if self.reduce == "allreduce":
            h = self._host(t.contiguous())
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
            if h is not t:
                t.copy_(h.to(t.device).view(t.shape))
            return t
        src = self._host(t.contiguous())
        parts = [torch.empty_like(src) for _ in range(self.size)]
        dist.all_gather(parts, src, group=self.group)
        if t.is_cuda:
            flat = t.view(-1, 1) if t.is_contiguous() else None
            acc = parts[0].to(t.device).reshape(-1, 1)
            for p in parts[1:]:
                D.axpby(dev, 1.0, p.to(t.device).reshape(-1, 1), 1.0, acc)
            if flat is not None:
                D.copy(dev, acc, flat)
            else:
                t.copy_(acc.view(t.shape))
            return t
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p
        t.copy_(acc)
        return t

    def broadcast(self, t, src=0):
        if self.size == 1:
            return t
        h = self._host(t.contiguous())
        dist.broadcast(h, src=src, group=self.group)
        if h is not t:
            t.copy_(h.to(t.device).view(t.shape))
        return t

    def exchange(self, sends, recvs):
        """Point-to-point: sends[q] -> rank q, recvs[q] <- rank q (None = nothing)."""
        ops = []
        staged_recv = []
        for q in range(self.size):
            if q == self.rank:
                continue
            if sends[q] is not None and sends[q].numel():
                ops.append(dist.P2POp(dist.isend, self._host(sends[q].contiguous()), q, self.group))
            if recvs[q] is not None and recvs[q].numel():
                buf = torch.empty(recvs[q].shape, dtype=recvs[q].dtype) if self.staged else recvs[q]
                staged_recv.append((buf, recvs[q]))
                ops.append(dist.P2POp(dist.irecv, buf, q, self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for buf, dst in staged_recv:
            if buf is not dst:
                dst.copy_(buf.to(dst.device))


class DistProblem:
    """This rank's share of A (and B) in HBM plus the halo plan."""

    def __init__(self, dev, part, comm, n_global, A=None, B=None):
        self.dev = self.ctx = dev
        self.part = part
        self.comm = comm
        self.n = part.nloc                      # rows owned (the solver's local n)
        self.n_global = n_global
        self.nghost = part.nghost
        if A is None:
            A = DeviceCsr.from_scipy(dev, part.a)
            if part.b is not None:
                B = A.with_values(dev.upload(part.b.data.astype(np.float64)))
        self.A = A
        self.A.n = part.nloc
        self.B = B
        self._shift_vals = None
        self._shift_theta = None
        send = [np.asarray(s, dtype=np.int32) for s in part.send_rows]
        self.send_counts = np.array([s.shape[0] for s in send], dtype=np.int64)
        self.send_offs = np.concatenate([[0], np.cumsum(self.send_counts)])
        self.recv_offs = np.concatenate([[0], np.cumsum(part.recv_counts)])
        self.nsend = int(self.send_offs[-1])
        allsend = np.concatenate(send) if self.nsend else np.zeros(1, dtype=np.int32)
        self.send_idx = dev.upload(allsend.astype(np.int32))

    def shifted(self, theta):
        """(values, diag_shift) of A - theta*B on the local rows (see DeviceProblem.shifted)."""
        return DeviceProblem.shifted(self, theta)

    def halo(self, X):
        """Refresh the ghost rows following the local block X (n_local x k view)."""
        k = X.shape[1]
        if self.comm.size == 1 or k == 0:
            return
        full = X.as_strided((self.n + self.nghost, k), X.stride())
        send = self.dev.empty(max(self.nsend, 1), k)
        if self.nsend:
            D.gather_rows(self.dev, self.send_idx[: self.nsend], X, send[: self.nsend])
        recv = self.dev.empty(max(self.nghost, 1), k)
        sends = [send[self.send_offs[q]:self.send_offs[q + 1]] if self.send_counts[q] else None
                 for q in range(self.comm.size)]
        recvs = [recv[self.recv_offs[q]:self.recv_offs[q + 1]] if self.part.recv_counts[q] else None
                 for q in range(self.comm.size)]
        self.comm.exchange(sends, recvs)
        if self.nghost:
            D.copy(self.dev, recv[: self.nghost], full[self.n:])


class DistOps(LocalOps):
    """Row-partitioned operations (one rank of a torch.distributed job)."""

    distributed = True

    def __init__(self, dev, prob):
        super().__init__(dev, prob)
        self.comm = prob.comm
        self.rank, self.size = self.comm.rank, self.comm.size
        self.nloc = prob.n
        self.nghost = prob.nghost
        self.n_global = prob.n_global
        self.row0 = prob.part.r0
        self._keep = []

    def spmm(self, op, X, Y, **kw):
        self.prob.halo(X)
        return D.spmm(self.dev, op, X, Y, **kw)

    def gram(self, X, Y, G, **kw):
        tmp = self.dev.empty(X.shape[1], Y.shape[1])
        D.gram(self.dev, X, Y, tmp)
        self.comm.allgather_sum(self.dev, tmp)
        alpha = kw.get("alpha", 1.0)
        beta = kw.get("beta", 0.0)
        if kw.get("transpose_out"):
            G = G.t()
        if alpha == 1.0 and beta == 0.0:
            G.copy_(tmp)
        else:
            G.mul_(beta).add_(tmp, alpha=alpha)
        return G

    def col_dots(self, X, Y, out):
        D.col_dots(self.dev, X, Y, out)
        self.comm.allgather_sum(self.dev, out)
        return out

    def residuals(self, AX, X, BX, lam, mode, out):
        sums = self.dev.empty(4 * X.shape[1])
        D.ritz_sums(self.dev, AX, X, BX, lam, mode, sums)
        self.comm.allgather_sum(self.dev, sums)
        return D.ritz_finish(self.dev, sums, lam, mode, out)

    def broadcast(self, t):
        return self.comm.broadcast(t, src=0)

    def allgather_sum_small(self, t):
        return self.comm.allgather_sum(self.dev, t)

    def _cg(self, vals, shift, rhs, x, max_iters, rel_tol, sweeps, conv, frozen, relres):
        k = rhs.shape[1]
        prob, comm, dev = self.prob, self.comm, self.dev
        send = dev.empty(max(prob.nsend, 1), k)
        recv = dev.empty(max(prob.nghost, 1), k)
        red = dev.empty(k)
        sends = [send[prob.send_offs[q]:prob.send_offs[q + 1]] if prob.send_counts[q] else None
                 for q in range(comm.size)]
        recvs = [recv[prob.recv_offs[q]:prob.recv_offs[q + 1]] if prob.part.recv_counts[q] else None
                 for q in range(comm.size)]

        def callback(op, kk, user):
            try:
                if op == 0:
                    comm.exchange(sends, recvs)
                else:
                    comm.allgather_sum(dev, red)
                return 0
            except Exception:  # never let an exception unwind through C
                return 1

        cb = _lib.CG_DIST_CALLBACK(callback)
        d = _lib.CgDist(prob.nghost, prob.nsend, C.c_void_p(prob.send_idx.data_ptr()),
                        C.c_void_p(send.data_ptr()), C.c_void_p(recv.data_ptr()),
                        C.c_void_p(red.data_ptr()), cb, None)
        keep = []
        if comm.native is not None:
            # the library exchanges the halo and sums the k-vectors itself (nccl.cu)
            peers = [q for q in range(comm.size) if q != comm.rank and
                     (prob.send_counts[q] or prob.part.recv_counts[q])]
            pr = (C.c_int32 * max(1, len(peers)))(*peers)
            so = (C.c_int64 * (len(peers) + 1))(*([int(prob.send_offs[q]) for q in peers] +
                                                  [int(prob.send_offs[peers[-1] + 1]) if peers else 0]))
            ro = (C.c_int64 * (len(peers) + 1))(*([int(prob.recv_offs[q]) for q in peers] +
                                                  [int(prob.recv_offs[peers[-1] + 1]) if peers else 0]))
            keep = [pr, so, ro]
            d.callback = _lib.CG_DIST_CALLBACK()
            d.nccl_comm = comm.native.handle
            d.npeer = len(peers)
            d.peer_rank = C.cast(pr, C.c_void_p)
            d.peer_send_off = C.cast(so, C.c_void_p)
            d.peer_recv_off = C.cast(ro, C.c_void_p)
        D.block_cg_dist(dev, prob.A, vals, shift, rhs, x, max_iters, rel_tol, sweeps, conv, frozen,
                        relres, d)
        del keep



def gcg_solve_distributed(a, b=None, config=None, *, comm=None, plane=1, x0=None, dev=None):
    """Row-partitioned `gcg_solve` for the calling rank of a torch.distributed job.

    Every rank passes the same global host matrices (or only needs the rows it
    owns plus their pattern — `local_part` slices them); rows are cut in blocks
    aligned to `plane` rows (one grid plane for the BASELINE stencils).  The
    report holds the global eigenvalues/residuals and this rank's rows of the
    eigenvectors (`report.row_range`).
    """
    from .solver import SolverConfig, gcg_solve_ops

    cfg = config if config is not None else SolverConfig()
    comm = comm if comm is not None else Comm()
    dev = dev if dev is not None else D.default_context()
    a = scipy.sparse.csr_matrix(a)
    n = a.shape[0]
    bounds = row_bounds(n, comm.size, plane)
    part = local_part(a, b, bounds, comm.rank)
    prob = DistProblem(dev, part, comm, n)
    return gcg_solve_ops(DistOps(dev, prob), cfg, x0=x0)
