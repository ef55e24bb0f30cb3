"""LIBSVM ingest (dataset.py:242-293): the native parser of
libsnx (host code, no GPU needed) + label remap + storage choice against the
reference's load_libsvm on the same files (tests/golden/libsvm/)."""

import numpy as np
import pytest

import paper_1802_09113_b200 as snx
from conftest import libsvm_cases
from paper_1802_09113_b200 import _build, io


@pytest.fixture(scope="module", autouse=True)
def _built():
    _build.build()  # the parser lives in libsnx (host code; no GPU needed)


def test_libsvm_matches_reference(libsvm_golden):
    seen = 0
    for name, path, C, nf, storage, g in libsvm_cases(libsvm_golden):
        err = str(g["error"])
        if err == "ParseError":
            with pytest.raises(snx.ParseError) as ei:
                io.parse_libsvm(path, C, nf)
            assert ei.value.line_number == int(g["line"]), name
        elif err == "DataError":
            with pytest.raises(snx.DataError):
                io.parse_libsvm(path, C, nf)
        else:
            csr, y = io.parse_libsvm(path, C, nf)
            assert np.array_equal(csr.toarray(), g["X"], equal_nan=True), name
            assert np.array_equal(y, g["y"]), name
            assert io.picks_dense(csr, storage) == (not bool(g["is_sparse"])), name
        seen += 1
    assert seen == 15  # incl. Python float()/int() token grammar: underscores, inf/nan, no hex


def test_libsvm_missing_file(tmp_path):
    with pytest.raises(OSError):
        io.read_libsvm(str(tmp_path / "nope.svm"))


def test_libsvm_large_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    n, p = 2000, 3000
    lines, rows = [], []
    for i in range(n):
        cols = np.sort(rng.choice(p, size=int(rng.integers(0, 40)), replace=False))
        vals = rng.standard_normal(len(cols))
        rows.append((cols, vals))
        lines.append(" ".join([str(i % 7)] + [f"{c + 1}:{float(v)!r}" for c, v in zip(cols, vals)]))
    path = tmp_path / "big.svm"
    path.write_text("\n".join(lines) + "\n")
    raw, indptr, indices, data, mx = io.read_libsvm(str(path))
    assert len(raw) == n and indptr[-1] == sum(len(c) for c, _ in rows)
    for i in (0, 17, n - 1):
        a, b = indptr[i], indptr[i + 1]
        assert np.array_equal(indices[a:b], rows[i][0])
        assert np.array_equal(data[a:b], rows[i][1])  # repr round trip: exact
