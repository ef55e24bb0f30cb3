"""GPU parity of the SURVEY 8(f) rows: estimate_lipschitz (bench.py:116-138),
normalize_columns / train_test_split (dataset.py:314-342) and the trace CSV
of a device solve, against the reference's golden vectors and the oracle."""

import os

import numpy as np
import pytest
import torch

import oracle
import paper_1802_09113_b200 as snx
from conftest import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _ds(A, y, C, dtype="f64"):
    return snx.DeviceDataset.from_numpy(A, y, C, dtype=dtype)


def _host(ds):
    return ds.X[:, :ds.n_features].double().cpu().numpy()


def test_lipschitz_golden(data_golden, solver_golden):
    g = data_golden
    for i in range(4):
        n, p, C, seed, iters = (int(t) for t in g[f"lp{i}_params"])
        prob = snx.SoftmaxProblem(_ds(g[f"lp{i}_A"], g[f"lp{i}_y"], C), 1e-3)
        L = snx.estimate_lipschitz(prob, iters=iters)
        ref = float(g[f"lp{i}_L"])
        if ref == 0.0:
            assert L == 0.0
        else:
            assert abs(L - ref) <= 1e-10 * abs(ref), (i, L, ref)
    s = solver_golden
    prob = snx.SoftmaxProblem(_ds(s["lip_A"], s["lip_y"], 3), 1e-3)
    L = snx.estimate_lipschitz(prob, iters=50)
    assert abs(L - float(s["lip_L"])) <= 1e-10 * float(s["lip_L"])
    assert snx.estimate_lipschitz(prob, iters=0) == 0.0


def test_lipschitz_f32_and_rerun():
    A, y = oracle.synthetic_problem(3000, 64, 10, seed=5)
    ref = oracle.estimate_lipschitz(A, y, 10, iters=100)
    p64 = snx.SoftmaxProblem(_ds(A, y, 10), 0.0)
    a, b = snx.estimate_lipschitz(p64, iters=100), snx.estimate_lipschitz(p64, iters=100)
    assert a == b  # fixed-order reductions: bit-identical reruns
    assert abs(a - ref) <= 1e-10 * ref
    L32 = snx.estimate_lipschitz(snx.SoftmaxProblem(_ds(A, y, 10, "f32"), 0.0), iters=100)
    assert abs(L32 - ref) <= 1e-4 * ref


def test_lipschitz_empty_raises():
    ds = _ds(np.zeros((0, 4)), np.zeros(0, dtype=np.int64), 3)
    with pytest.raises(snx.DataError):
        snx.estimate_lipschitz(snx.SoftmaxProblem(ds, 1e-3))


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_normalize_columns_golden(data_golden, dtype):
    g = data_golden
    for i in range(3):
        A, y, C = g[f"nc{i}_A"], g[f"nc{i}_y"], int(g[f"nc{i}_C"])
        ds = _ds(A, y, C, dtype)
        norms, _ = snx.column_norms(ds)
        out = snx.normalize_columns(ds)
        assert out is not ds and out.n_rows == ds.n_rows
        tol = 1e-14 if dtype == "f64" else 1e-6
        ref_n = g[f"nc{i}_norms"]
        if dtype == "f64":
            assert rel_err(norms.cpu().numpy(), ref_n) <= tol
            assert rel_err(_host(out), g[f"nc{i}_A_norm"]) <= tol
        got = _host(out)
        nz = ref_n > 0
        if dtype == "f32":  # tiny columns underflow in f32: compare the normal ones
            nz &= ref_n > 1e-30
            assert rel_err(got[:, nz], g[f"nc{i}_A_norm"][:, nz]) <= tol
        assert np.all(got[:, ~(ref_n > 0)] == 0.0)  # zero columns untouched
        assert np.array_equal(_host(ds), A.astype(np.float32 if dtype == "f32" else np.float64))
        if ds.ld > ds.n_features:  # pad columns stay zero
            assert float(out.X[:, ds.n_features:].abs().sum()) == 0.0


def test_normalize_columns_cifar_shape():
    gen = np.random.default_rng(3)
    A = gen.standard_normal((20000, 3072)) * gen.uniform(0.1, 10.0, 3072)
    y = gen.integers(0, 10, 20000)
    ds = _ds(A, y, 10)
    out = _host(snx.normalize_columns(ds))
    assert rel_err(out, oracle.normalize_columns(A)) <= 1e-14
    assert np.allclose(np.linalg.norm(out, axis=0), 1.0, rtol=1e-13, atol=0)


def test_train_test_split_golden(data_golden):
    g = data_golden
    for i in range(4):
        n, f, seed = g[f"sp{i}_params"]
        n = int(n)
        A = np.zeros((n, 2))
        A[:, 0] = np.arange(n)
        ds = _ds(A, np.arange(n) % 2, 2)
        tr, te = snx.train_test_split(ds, float(f), int(seed))
        assert np.array_equal(_host(tr.materialized())[:, 0].astype(np.int64), g[f"sp{i}_train"])
        assert np.array_equal(_host(te.materialized())[:, 0].astype(np.int64), g[f"sp{i}_test"])
    with pytest.raises(snx.DataError):
        snx.train_test_split(ds, 1.0, 0)
    one = _ds(np.zeros((1, 2)), np.zeros(1, dtype=np.int64), 2)
    with pytest.raises(snx.DataError):
        snx.train_test_split(one, 0.5, 0)


def test_prepare_then_solve_trace_csv(tmp_path):
    """The reference's prepare_data (bench.py:149-155: normalise, split) on the
    device, a Newton solve with a test set, and its trace CSV."""
    gen = np.random.default_rng(9)
    A = gen.standard_normal((3000, 40)) * gen.uniform(0.5, 5.0, 40)
    y = gen.integers(0, 5, 3000)
    ds = snx.normalize_columns(_ds(A, y, 5))
    train, test = snx.train_test_split(ds, 0.8, 4)
    An = oracle.normalize_columns(A)
    tr_idx, te_idx = oracle.train_test_split(3000, 0.8, 4)
    cfg = snx.make_variant("subsampled-100", snx.NewtonConfig(max_outer_iters=5))
    paths = []
    for rerun in range(2):
        tr = snx.newton_solve(snx.SoftmaxProblem(train.materialized(), 1e-3), cfg,
                              test_set=test.materialized())
        for r in tr.records:
            r.cum_seconds = 0.0
        paths.append(os.path.join(tmp_path, f"t{rerun}.csv"))
        snx.write_trace_csv(paths[-1], tr.records)
    with open(paths[0], "rb") as a, open(paths[1], "rb") as b:
        assert a.read() == b.read()  # reruns byte-identical (tests/test_acceptance.py:316-348)
    ref = oracle.newton_solve(An[tr_idx], y[tr_idx], 5, 1e-3, "subsampled-100",
                              max_outer_iters=5, test=(An[te_idx], y[te_idx]))
    back = snx.read_trace_csv(paths[0])
    assert [r.iteration for r in back] == [int(r[0]) for r in ref["records"]]
    assert np.allclose([r.objective for r in back], [r[1] for r in ref["records"]],
                       rtol=1e-10, atol=0)
    assert [r.test_acc for r in back] == [r[3] for r in ref["records"]]
