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
