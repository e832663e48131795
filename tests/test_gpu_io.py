"""History / RunRecord output of a device solve (reference test_io.py:268-342), plus a
MatrixMarket file solved end to end."""

import json

import numpy as np
import pytest

from paper_2111_06552_b200 import (
    IoError,
    RunRecord,
    SolverConfig,
    Unsupported,
    gcg_solve,
    history_rows,
    read_matrix_market,
    write_history,
    write_matrix_market,
)
from paper_2111_06552_b200 import problems as P
from paper_2111_06552_b200.io import HISTORY_COLUMNS

pytestmark = pytest.mark.gpu


def _small_report(**over):
    cfg = SolverConfig(num_eigen=2, tol=1e-9, seed=1, **over)
    return gcg_solve(np.diag(np.arange(1.0, 11.0)), config=cfg)


def test_history_csv_shape(tmp_path):
    rep = _small_report()
    path = tmp_path / "h.csv"
    write_history(rep, str(path))
    lines = path.read_text().strip().splitlines()
    assert lines[0] == ",".join(HISTORY_COLUMNS)
    assert len(lines) == 1 + rep.iterations
    first = lines[1].split(",")
    assert len(first) == len(HISTORY_COLUMNS) and first[0] == "1"


def test_history_empty_gives_header_only(tmp_path):
    rep = _small_report(collect_history=False)
    assert rep.history == []
    path = tmp_path / "h.csv"
    write_history(rep, str(path))
    assert path.read_text() == ",".join(HISTORY_COLUMNS) + "\n"


def test_history_json_and_csv_agree(tmp_path):
    rep = _small_report()
    cpath, jpath = tmp_path / "h.csv", tmp_path / "h.json"
    write_history(rep, str(cpath))
    write_history(rep, str(jpath), format="json")
    rows = json.loads(jpath.read_text())
    lines = cpath.read_text().strip().splitlines()
    assert len(rows) == len(lines) - 1
    for row, line in zip(rows, lines[1:]):
        for col, cell in zip(HISTORY_COLUMNS, line.split(",")):
            assert float(cell) == row[col]


def test_history_errors(tmp_path):
    rep = _small_report()
    with pytest.raises(Unsupported):
        write_history(rep, str(tmp_path / "h.xml"), format="xml")
    with pytest.raises(IoError):
        write_history(rep, str(tmp_path / "no" / "dir" / "h.csv"))


def test_step_timings_are_gpu_time():
    """t_step* come from CUDA events: non-negative, and STEP 6 (block CG) is nonzero."""
    pr = P.baseline_problem(1)
    rep = gcg_solve(pr.a, None, SolverConfig(num_eigen=20, block_size=20, tol=1e-8, seed=0))
    t6 = [h.timings["t_step6"] for h in rep.history]
    assert all(v >= 0.0 for h in rep.history for v in h.timings.values())
    assert sum(t6) > 0.0


def test_run_record_roundtrip():
    rep = _small_report()
    config = {"num_eigen": 2, "tol": 1e-9, "deterministic": False}
    rec = RunRecord.from_run(rep, config, wall_time=1.25, nnz_a=10)
    back = RunRecord.from_json(rec.to_json())
    assert back == rec
    assert rec.schema_version == 1 and rec.backend == "sm100"
    assert rec.nnz_a == 10 and rec.nnz_b is None and rec.wall_time == 1.25
    assert rec.history == history_rows(rep)
    assert len(rec.eigenvalues) == 2
    assert np.asarray(rec.eigenvectors).shape == (10, 2)


def test_run_record_deterministic_zeroes_clocks(tmp_path):
    """Deterministic runs serialise to identical bytes (test_acceptance.py:322-342)."""
    texts = []
    for k in range(2):
        rep = _small_report(deterministic=True)
        rec = RunRecord.from_run(rep, {"num_eigen": 2, "deterministic": True}, wall_time=3.0 + k)
        assert rec.wall_time == 0.0
        assert all(v == 0.0 for v in rec.timings.values())
        path = tmp_path / f"r{k}.json"
        rec.write(str(path))
        texts.append(path.read_text())
    assert texts[0] == texts[1]


def test_matrix_market_file_solved_end_to_end(tmp_path):
    """write -> native read -> solve: the 2-D Laplacian's analytic spectrum."""
    pr = P.baseline_problem(1)
    path = str(tmp_path / "lap2d.mtx")
    write_matrix_market(pr.a, path)
    a = read_matrix_market(path)
    assert (a != pr.a.tocsr()).nnz == 0
    rep = gcg_solve(a, None, SolverConfig(num_eigen=20, block_size=20, tol=1e-8, seed=0,
                                          init="normal", residual="relative"))
    exact = P.analytic_eigenvalues(1, 20)
    assert rep.status == "converged"
    assert np.abs(rep.eigenvalues - exact).max() / exact.max() <= 1e-9


def _mm_text(path, header, size, entries):
    with open(path, "w") as fh:
        fh.write(header + "\n% a comment\n" + size + "\n")
        for e in entries:
            fh.write(e + "\n")


@pytest.mark.parametrize("case", ["general", "symmetric", "duplicates", "empty_rows", "lap3d"])
def test_device_matrix_market_ingestion(tmp_path, case):
    """read_matrix_market_device (native tokeniser + device COO->CSR: stable radix sort,
    duplicate sums, scanned row pointers) equals the host reader; bit for bit without
    duplicate entries."""
    import scipy.sparse

    from paper_2111_06552_b200 import device as D
    from paper_2111_06552_b200.io import read_matrix_market, read_matrix_market_device, \
        write_matrix_market

    p = tmp_path / f"{case}.mtx"
    rng = np.random.default_rng(3)
    if case == "general":
        m = scipy.sparse.random(300, 300, density=0.03, random_state=5, format="csr")
        m = m + m.T + scipy.sparse.eye(300)
        write_matrix_market(m, p)
    elif case == "symmetric":
        ents = [f"{i} {i} {4.0 + i / 7}" for i in range(1, 51)] + \
               [f"{i + 1} {i} {-1.0 - i / 13}" for i in range(1, 50)]
        _mm_text(p, "%%MatrixMarket matrix coordinate real symmetric", f"50 50 {len(ents)}", ents)
    elif case == "duplicates":
        ents = [f"{i} {i} 1.5" for i in range(1, 41)] + ["3 4 0.1", "4 3 0.1", "3 4 0.2",
                                                          "4 3 0.2", "3 4 1e-17", "4 3 1e-17"]
        rng.shuffle(ents)
        _mm_text(p, "%%MatrixMarket matrix coordinate real general", f"40 40 {len(ents)}", ents)
    elif case == "empty_rows":
        ents = ["1 1 2.0", "7 7 3.0", "7 2 -1.0", "2 7 -1.0", "30 30 1.0"]
        _mm_text(p, "%%MatrixMarket matrix coordinate real general", f"30 30 {len(ents)}", ents)
    else:
        write_matrix_market(P.laplacian_3d(12), p)
    host = read_matrix_market(p)
    dev = D.default_context()
    d = read_matrix_market_device(p, dev)
    assert d.n == host.shape[0] and d.nnz == host.nnz
    assert np.array_equal(d.rowptr.cpu().numpy(), host.indptr)
    assert np.array_equal(d.colidx.cpu().numpy(), host.indices)
    if case == "duplicates":
        assert np.allclose(d.val.cpu().numpy(), host.data, rtol=1e-15, atol=0)
    else:
        assert np.array_equal(d.val.cpu().numpy(), host.data)


def test_device_matrix_market_errors_match_host(tmp_path):
    """Malformed files raise the reference's errors before any device work."""
    from paper_2111_06552_b200.errors import ParseError
    from paper_2111_06552_b200.io import read_matrix_market_device

    p = tmp_path / "bad.mtx"
    _mm_text(p, "%%MatrixMarket matrix coordinate real general", "3 3 2", ["1 1 1.0", "4 1 2.0"])
    with pytest.raises(ParseError) as e:
        read_matrix_market_device(p)
    assert e.value.line == 5
