"""Alg. 2 (modified_block_orth) on the B200 against the reference's own run.

The golden vectors (tests/golden/golden_alg2.npz) come from the unmodified
reference on the test_orth.py shapes; decisions (kept columns, replaced slots,
reduction counts m + m/b - 1) must match exactly, the orthonormalised block to
rounding level, and the Gram defect must meet the reference's bound
(test_orth.py:46-67, 94-107, 145-178).
"""

import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import scipy.sparse
import torch

from paper_2111_06552_b200 import OrthConfig, modified_block_orth
from paper_2111_06552_b200 import device as D
from paper_2111_06552_b200.errors import AllDependent
from paper_2111_06552_b200.operators import DeviceCsr
from tests.conftest import ALG2_KW, ALG2_TAGS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    return D.default_context()


def _b_for(tag, n):
    if tag != "with_b":
        return None
    return scipy.sparse.diags([np.ones(n - 1), 4.0 * np.ones(n), np.ones(n - 1)], [-1, 0, 1],
                              format="csr")


@pytest.mark.parametrize("tag", ALG2_TAGS)
def test_alg2_matches_reference(dev, golden_alg2, tag):
    g = golden_alg2
    xin = g[f"{tag}_in"]
    n = xin.shape[0]
    bs = _b_for(tag, n)
    b = DeviceCsr.from_scipy(dev, bs) if bs is not None else None
    x = torch.from_numpy(np.ascontiguousarray(xin)).to(dev.device)
    x0 = None
    if f"{tag}_x0" in g:
        x0 = torch.from_numpy(np.ascontiguousarray(g[f"{tag}_x0"])).to(dev.device)
    out = modified_block_orth(dev, x, x0=x0, b=b, cfg=OrthConfig(**ALG2_KW[tag]))
    kept, red = (int(v) for v in g[f"{tag}_meta"])
    assert (out.num_kept, out.reduction_count) == (kept, red)
    assert out.replaced_indices == [int(v) for v in g[f"{tag}_replaced"]]
    got = x.cpu().numpy()[:, :kept]
    want = g[f"{tag}_out"][:, :kept]
    assert np.abs(got - want).max() <= 1e-10
    bx = got if bs is None else bs @ got
    assert np.abs(got.T @ bx - np.eye(kept)).max() <= 1e-9


def test_alg2_all_dependent_raises(dev):
    with pytest.raises(AllDependent):
        modified_block_orth(dev, dev.zeros(20, 4))


def test_alg2_idempotent_on_orthonormal_input(dev):
    """test_orth.py:121-127: a second pass changes nothing beyond rounding."""
    rng = np.random.default_rng(11)
    x = torch.from_numpy(rng.uniform(-1, 1, (40, 6))).to(dev.device)
    modified_block_orth(dev, x)
    before = x.clone()
    out = modified_block_orth(dev, x)
    assert out.num_kept == 6
    assert float((x - before).abs().max()) <= 1e-12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2111_06552_b200.distributed import Comm, DistOps, row_bounds

        g = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_alg2.npz"))
        xin = g["m96_b16_in"]
        n = xin.shape[0]
        cuts = row_bounds(n, world)
        r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
        dev = D.default_context()
        prob = SimpleNamespace(comm=Comm(), n=r1 - r0, nghost=0, n_global=n,
                               part=SimpleNamespace(r0=r0), B=None)
        ops = DistOps(dev, prob)
        x = torch.from_numpy(np.ascontiguousarray(xin[r0:r1])).to(dev.device)
        out = modified_block_orth(ops, x, cfg=OrthConfig(block_width=16))
        q.put((rank, out.num_kept, out.reduction_count, r0, x.cpu().numpy()))
    except Exception as exc:  # report instead of hanging the parent
        q.put((rank, "error", repr(exc), None, None))
    finally:
        dist.destroy_process_group()


def test_alg2_two_ranks(golden_alg2):
    """Row-partitioned Alg. 2: every reduction is one ordered all-gather sum."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        item = q.get(timeout=300)
        res[item[0]] = item
    for p in procs:
        p.join(timeout=60)
    kept, red = (int(v) for v in golden_alg2["m96_b16_meta"])
    for r in (0, 1):
        assert res[r][1:3] == (kept, red), res[r][:3]
    full = np.concatenate([res[0][4], res[1][4]])
    assert np.abs(full - golden_alg2["m96_b16_out"]).max() <= 1e-10


# ---- native (C++) Alg. 3 driver vs the Python control flow -----------------------------


def _run_both(dev, fn, *host_arrays):
    """Run `fn(native: bool) -> (outcome, result arrays)` with the native driver on and off."""
    from paper_2111_06552_b200 import orth as O

    saved = O._NATIVE
    try:
        O._NATIVE = True
        a = fn()
        O._NATIVE = False
        b = fn()
    finally:
        O._NATIVE = saved
    return a, b


@pytest.mark.parametrize("case", ["strict", "default", "against", "against_b", "dependent"])
def test_native_orth_matches_python_driver(dev, golden, case):
    from paper_2111_06552_b200 import orth_against, recursive_orth_svd

    def blk(n, m, seed):
        return np.random.default_rng(seed).uniform(-1, 1, (n, m))

    b = None
    if case in ("strict", "default"):
        xin, basis = golden[f"orth_{case}_in"], None
        cfg = OrthConfig(reorth_tol=1e-15 if case == "strict" else 1e-10)
    elif case == "against":
        xin, basis, cfg = golden["oa_in"], golden["oa_basis"], OrthConfig()
    elif case == "against_b":
        n = 300
        bs = _b_for("with_b", n)
        b = DeviceCsr.from_scipy(dev, bs)
        basis = blk(n, 12, 5)
        bt = torch.from_numpy(basis).to(dev.device)
        recursive_orth_svd(dev, bt, b=b)
        basis = bt.cpu().numpy()
        xin, cfg = blk(n, 20, 6), OrthConfig()
    else:
        xin = blk(200, 24, 7)
        xin[:, 5] = xin[:, 2]
        xin[:, 17] = 0.0
        basis, cfg = None, OrthConfig()

    def run():
        x = torch.from_numpy(np.ascontiguousarray(xin)).to(dev.device)
        if basis is None:
            out = recursive_orth_svd(dev, x, b=b, cfg=cfg)
        else:
            out = orth_against(dev, x, torch.from_numpy(np.ascontiguousarray(basis)).to(dev.device),
                               b=b, cfg=cfg)
        return out, x.cpu().numpy()

    (oa, xa), (ob, xb) = _run_both(dev, run)
    assert (oa.num_kept, oa.reduction_count, oa.replaced_indices) == \
        (ob.num_kept, ob.reduction_count, ob.replaced_indices)
    k = oa.num_kept
    assert np.abs(xa[:, :k] - xb[:, :k]).max() <= 1e-12
