"""MatrixMarket ingestion (native parser) and the builtin generators — host side, no GPU.

Cases follow the reference's test_io.py (error line numbers, unsupported
headers, comments/blank lines, array format, round trip) and cross-check the
parsed matrices against scipy.io.mmread on random files.
"""

import io as _stdio
import math

import numpy as np
import pytest
import scipy.io
import scipy.sparse

from paper_2111_06552_b200 import (
    InvalidShape,
    IoError,
    ParseError,
    UnknownGenerator,
    Unsupported,
    generate_builtin,
    read_matrix_market,
    write_matrix_market,
)
from paper_2111_06552_b200.io import GENERATOR_NAMES


def _write(tmp_path, text, name="m.mtx"):
    path = tmp_path / name
    path.write_text(text)
    return str(path)


@pytest.mark.parametrize(
    "text,line",
    [
        ("%%MatrixMarket matrix coordinate real\n1 1 0\n", 1),
        ("not a banner\n1 1 0\n", 1),
        ("%%MatrixMarket matrix coordinate real general\n2 2\n", 2),
        ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n", 3),
        ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", 3),
        ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 abc\n", 3),
        ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", 4),
        ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 1.0\n", 4),
        ("%%MatrixMarket matrix array real general\n2 2\n1.0\n2.0\n3.0\n", 6),
        ("", 1),
        ("%%MatrixMarket matrix coordinate real general\n% only comments\n\n", 4),
        ("%%MatrixMarket matrix coordinate real general\n2 2 -1\n", 2),
        ("%%MatrixMarket matrix coordinate real general\n2 x 1\n1 1 1\n", 2),
        ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0 4\n", 3),
        ("%%MatrixMarket matrix array real symmetric\n2 3\n1\n2\n3\n", 2),
        ("%%MatrixMarket matrix array real general\n1 2\n1.0 2.0 3.0\n", 3),
        ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 0x1p3\n", 3),
    ],
)
def test_parse_errors_carry_line_numbers(tmp_path, text, line):
    with pytest.raises(ParseError) as exc:
        read_matrix_market(_write(tmp_path, text))
    assert exc.value.line == line
    assert f"line {line}:" in str(exc.value)


def test_first_error_in_file_order_across_threads(tmp_path):
    """Thousands of entry lines split over many parser threads: the malformed line wins
    over a later surplus, and a surplus before a malformed line wins over it."""
    n = 40000
    body = "".join(f"{i % 50 + 1} {i % 37 + 1} {i * 0.5}\n" for i in range(n))
    bad = body.splitlines(keepends=True)
    bad[30000] = "1 1 nan-ish\n"
    text = f"%%MatrixMarket matrix coordinate real general\n50 50 {n}\n" + "".join(bad)
    with pytest.raises(ParseError) as exc:
        read_matrix_market(_write(tmp_path, text), nthreads=8)
    assert exc.value.line == 30000 + 3
    text = f"%%MatrixMarket matrix coordinate real general\n50 50 {n - 15000}\n" + "".join(bad)
    with pytest.raises(ParseError) as exc:
        read_matrix_market(_write(tmp_path, text), nthreads=8)
    assert exc.value.line == n - 15000 + 3
    assert "more than the declared" in str(exc.value)


@pytest.mark.parametrize(
    "banner",
    [
        "%%MatrixMarket matrix coordinate complex general",
        "%%MatrixMarket matrix coordinate pattern general",
        "%%MatrixMarket matrix coordinate integer general",
        "%%MatrixMarket matrix coordinate real hermitian",
        "%%MatrixMarket matrix coordinate real skew-symmetric",
        "%%MatrixMarket vector coordinate real general",
    ],
)
def test_unsupported_headers(tmp_path, banner):
    with pytest.raises(Unsupported):
        read_matrix_market(_write(tmp_path, banner + "\n1 1 0\n"))


def test_missing_file_raises_io_error(tmp_path):
    with pytest.raises(IoError):
        read_matrix_market(str(tmp_path / "nope.mtx"))


def test_banner_is_case_insensitive_and_crlf(tmp_path):
    path = _write(tmp_path, "%%matrixmarket MATRIX Coordinate Real General\r\n1 1 1\r\n1 1 7.0\r\n")
    assert np.array_equal(read_matrix_market(path).toarray(), [[7.0]])


def test_comments_blank_lines_duplicates_and_order(tmp_path):
    path = _write(tmp_path, "%%MatrixMarket matrix coordinate real general\n% c\n\n2 2 4\n"
                            "2 2 5.0\n% between\n1 1 4.0\n1 2 0.0\n2 2 1.5\n")
    sp = read_matrix_market(path)
    assert np.array_equal(sp.toarray(), [[4.0, 0.0], [0.0, 6.5]])
    for i in range(2):
        row = sp.indices[sp.indptr[i]:sp.indptr[i + 1]]
        assert np.all(np.diff(row) > 0)


def test_array_format_general_and_symmetric(tmp_path):
    gen = _write(tmp_path, "%%MatrixMarket matrix array real general\n2 2\n1.0\n2.0\n2.0\n5.0\n",
                 name="g.mtx")
    assert np.array_equal(read_matrix_market(gen).toarray(), [[1.0, 2.0], [2.0, 5.0]])
    sym = _write(tmp_path, "%%MatrixMarket matrix array real symmetric\n2 2\n1.0\n2.0\n5.0\n",
                 name="s.mtx")
    assert np.array_equal(read_matrix_market(sym).toarray(), [[1.0, 2.0], [2.0, 5.0]])
    rect = _write(tmp_path, "%%MatrixMarket matrix array real general\n2 3\n1 2 3 4 5 6\n",
                  name="r.mtx")
    assert np.array_equal(read_matrix_market(rect).toarray(), [[1, 3, 5], [2, 4, 6]])


@pytest.mark.parametrize("sym", [False, True])
@pytest.mark.parametrize("n,density", [(9, 0.3), (400, 0.02), (3000, 0.004)])
def test_matches_scipy_mmread(tmp_path, sym, n, density):
    rng = np.random.default_rng(n)
    m = scipy.sparse.random(n, n, density=density, random_state=np.random.RandomState(n))
    m.data[:] = rng.standard_normal(m.nnz)
    m = (m + m.T).tocsr()
    path = str(tmp_path / "x.mtx")
    scipy.io.mmwrite(path, m, symmetry="symmetric" if sym else "general", precision=17)
    got = read_matrix_market(path, nthreads=4)
    want = scipy.io.mmread(path).tocsr()
    assert (got != want).nnz == 0
    assert got.shape == want.shape


def test_roundtrip_write_then_read(tmp_path):
    rng = np.random.default_rng(11)
    m = scipy.sparse.random(9, 9, density=0.3, random_state=np.random.RandomState(4))
    m.data[:] = rng.standard_normal(m.nnz)
    m = ((m + m.T) * 0.5).tocsr()
    path = tmp_path / "rt.mtx"
    write_matrix_market(m, str(path))
    back = read_matrix_market(str(path))
    assert np.array_equal(back.toarray(), m.toarray())


def test_write_unwritable_path(tmp_path):
    with pytest.raises(IoError):
        write_matrix_market(scipy.sparse.eye(3), str(tmp_path / "no" / "dir" / "m.mtx"))


# ---- generators (io.py:250-336; test_io.py generator cases) ----------------------


def test_laplacian1d_spectrum_and_entries():
    a, b = generate_builtin("laplacian1d", 3)
    assert b is None
    vals = np.linalg.eigvalsh(a.toarray())
    assert np.abs(vals - [2 - math.sqrt(2), 2, 2 + math.sqrt(2)]).max() <= 1e-14
    d = generate_builtin("laplacian1d", 5)[0].toarray()
    assert np.all(np.diag(d) == 2.0) and np.all(np.diag(d, 1) == -1.0)
    assert np.count_nonzero(d) == 5 + 2 * 4


def test_fem1d_pair():
    n = 7
    a, b = generate_builtin("fem1d-p1", n)
    h = 1.0 / (n + 1)
    assert np.allclose(np.diag(a.toarray()), 2.0 / h)
    assert np.allclose(np.diag(b.toarray()), 4.0 * h / 6.0)
    assert np.allclose(np.diag(b.toarray(), 1), h / 6.0)


def test_diag_range_and_clustered_random():
    a, _ = generate_builtin("diag-range", 6)
    assert np.array_equal(a.diagonal(), np.arange(1.0, 7.0))
    c, _ = generate_builtin("clustered-random", 64, density=0.05, seed=3)
    d = c.toarray()
    assert np.allclose(d, d.T)
    vals = np.linalg.eigvalsh(d)
    assert vals.min() > 0.0
    c2, _ = generate_builtin("clustered-random", 64, density=0.05, seed=3)
    assert (c != c2).nnz == 0  # seeded: identical


def test_generator_errors():
    with pytest.raises(UnknownGenerator):
        generate_builtin("nope", 5)
    with pytest.raises(InvalidShape):
        generate_builtin("laplacian1d", 1)
    assert GENERATOR_NAMES == tuple(sorted(GENERATOR_NAMES))
