"""Experiment harness: CSV ingest (dataset.py:296-311) and the
summary CSV writer (bench.py:36-46, 243-267) against fixtures the unmodified
reference produced (tests/golden/make_golden.py harness_golden)."""

import os
import tempfile

import numpy as np
import pytest

import paper_1802_09113_b200 as snx
from conftest import GOLDEN, load_golden
from paper_1802_09113_b200 import harness, io
from paper_1802_09113_b200.trace import RunRecord, SolveTrace


@pytest.fixture(scope="module")
def g():
    return load_golden("harness_golden.npz")


def csv_cases(g):
    for k in sorted(g):
        if k.startswith("csv_") and k.endswith("_C"):
            name = k[4:-2]
            yield name, os.path.join(GOLDEN, "csv", name + ".csv"), int(g[k]), {
                kk[len(f"csv_{name}_"):]: v for kk, v in g.items() if kk.startswith(f"csv_{name}_")}


def test_parse_csv_matches_reference(g):
    seen = 0
    for name, path, C, ref in csv_cases(g):
        err = str(ref["error"])
        if err == "ParseError":
            with pytest.raises(snx.ParseError):
                io.parse_csv(path, C)
        elif err == "DataError":
            with pytest.raises(snx.DataError):
                io.parse_csv(path, C)
        else:
            X, y = io.parse_csv(path, C)
            assert tuple(X.shape) == tuple(ref["shape"]), name
            assert np.array_equal(X, ref["X"]), name
            assert np.array_equal(y, ref["y"]), name
            assert y.dtype == np.int64
        seen += 1
    assert seen == 8  # empty file, ragged / bad numbers, too many labels, ...


def _traces():
    def trace(rows, reason):
        return SolveTrace(records=[RunRecord(*r) for r in rows], reason=reason)

    t1 = trace([("full-newton", 0, 0.0, 69.31471805599453, 0.25, float("nan"), 0.0, 0),
                ("full-newton", 1, 0.5, 12.000000000000002, 0.75, 0.5, 1.0, 7),
                ("full-newton", 2, 1.25, 11.5, 0.8, 0.625, 0.5, 10)], "gradient-converged")
    t2 = trace([("adam_lr0.1", 0, 0.0, 5.0, 0.1, 0.2, 0.0, 0),
                ("adam_lr0.1", 1, 0.75, float("inf"), 0.1, float("nan"), 0.0, 0)], "diverged")
    return [harness.RunResult("full-newton", "full-newton", None, t1),
            harness.RunResult("adam_lr0.1", "adam", 0.1, t2, classification="diverged"),
            harness.RunResult("rmsprop_lr3.5e-05", "rmsprop", 3.5e-05, t1,
                              classification="progressed")]


def test_summary_csv_byte_identical(g):
    results = _traces()
    for i, target in enumerate((None, 0.6, 0.99)):
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "summary.csv")
            harness.write_summary_csv(path, results, target)
            with open(path, "rb") as fh:
                assert fh.read() == bytes(g[f"summary{i}_bytes"]), target


def test_summary_schema_and_newton_config():
    assert harness.SUMMARY_COLUMNS[0] == "solver" and len(harness.SUMMARY_COLUMNS) == 9

    class Run:  # the reference's SolverRun, duck-typed
        method, epochs, epsilon, cg_tol, cg_max_iters, seed = "subnewton-20", 7, 1e-6, 1e-3, 12, 4

    cfg = harness.newton_config(Run())
    assert cfg.max_outer_iters == 7 and cfg.epsilon == 1e-6
    assert cfg.cg.theta == 1e-3 and cfg.cg.max_iters == 12 and cfg.samples.seed == 4
    assert cfg.samples.gradient_fraction == snx.VARIANT_FRACTIONS["subsampled-20"][0]

    class Adam(Run):
        method = "adam"

    with pytest.raises(ValueError):
        harness.execute_run(None, None, Adam())
    sent = []
    hook = harness.make_execute_run(lambda prob, test, run, learning_rate=None: sent.append(
        (run.method, learning_rate)) or "ref")
    assert hook(None, None, Adam(), learning_rate=0.1) == "ref" and sent == [("adam", 0.1)]
