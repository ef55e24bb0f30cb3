"""CPU side of the data-preparation / Lipschitz / trace-CSV rows:
the oracle restatements against the reference's golden vectors, and the
host-only trace CSV writer/reader against the reference's bytes."""

import os

import numpy as np

import oracle
from paper_1802_09113_b200 import trace


def test_normalize_columns_oracle(data_golden):
    g = data_golden
    i = 0
    while f"nc{i}_A" in g:
        A = g[f"nc{i}_A"]
        assert np.array_equal(oracle.column_norms(A), g[f"nc{i}_norms"])
        assert np.array_equal(oracle.normalize_columns(A), g[f"nc{i}_A_norm"])
        i += 1
    assert i == 3


def test_train_test_split_oracle(data_golden):
    g = data_golden
    for i in range(4):
        n, f, seed = g[f"sp{i}_params"]
        tr, te = oracle.train_test_split(int(n), float(f), int(seed))
        assert np.array_equal(tr, g[f"sp{i}_train"])
        assert np.array_equal(te, g[f"sp{i}_test"])


def test_lipschitz_oracle(data_golden):
    g = data_golden
    for i in range(4):
        n, p, C, seed, iters = (int(t) for t in g[f"lp{i}_params"])
        L = oracle.estimate_lipschitz(g[f"lp{i}_A"], g[f"lp{i}_y"], C, iters=iters)
        ref = float(g[f"lp{i}_L"])
        assert abs(L - ref) <= 1e-12 * max(abs(ref), 1e-300), (i, L, ref)


def _records():
    R = trace.RunRecord
    return [R("subsampled-100", 0, 0.0, 69.31471805599453, 0.25, float("nan"), 0.0, 0),
            R("subsampled-100", 1, 0.125, 41.00000000000001, 0.5, 0.3333333333333333, 1.0, 10),
            R("full", 2, 1e-300, float("inf"), 1.0, 0.1, 0.0625, 3)]


def test_trace_csv_bytes(data_golden, tmp_path):
    path = os.path.join(tmp_path, "t.csv")
    trace.write_trace_csv(path, _records())
    with open(path, "rb") as fh:
        assert fh.read() == bytes(data_golden["csv_bytes"])


def test_trace_csv_round_trip(tmp_path):
    path = os.path.join(tmp_path, "t.csv")
    recs = _records()
    trace.write_trace_csv(path, recs)
    back = trace.read_trace_csv(path)
    assert len(back) == len(recs)
    for a, b in zip(back, recs):
        assert a.as_row() == b.as_row()
    with open(path, "w") as fh:
        fh.write("a,b\n")
    try:
        trace.read_trace_csv(path)
    except ValueError:
        pass
    else:
        raise AssertionError("foreign header accepted")
