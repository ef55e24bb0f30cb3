"""CSR storage on the GPU (the reference's sparse DesignMatrix,
dataset.py:21-147) against the reference's own sparse results: fp64, 1e-10
relative, Newton traces with identical CG counts and step sizes."""

import numpy as np
import pytest
import scipy.sparse as sp
import torch

import oracle
import paper_1802_09113_b200 as snx
from conftest import rel_err, sparse_cases
from paper_1802_09113_b200.sparse import CsrDataset

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_sparse_golden(sparse_golden):
    for i, A, C, c in sparse_cases(sparse_golden):
        y, x, v = c["y"], c["x"], c["v"]
        ds = CsrDataset.from_scipy(A, y, C)
        prob = snx.SoftmaxProblem(ds, 1e-3)
        f = snx.objective(prob, x)
        assert abs(f - float(c["objective"])) <= TOL * abs(float(c["objective"])), i
        assert rel_err(snx.gradient(prob, x), c["gradient"]) <= TOL, i
        op = snx.HessianOperator(ds, x, 1e-3, scale=3.0)
        assert rel_err(op.apply(v), c["hess_apply"]) <= TOL, i
        assert snx.accuracy(ds, x) == float(c["accuracy"]), i
        seed = [71, 72, 73, 74][i]
        orc = snx.SubsampledOracle(prob, snx.SampleConfig(0.5, 0.1, False, seed), 2)
        assert rel_err(orc.gradient(x), c["orc_grad"]) <= TOL, i
        assert rel_err(orc.hess_vec(x, v), c["orc_hv"]) <= TOL, i
        rep = snx.SubsampledOracle(prob, snx.SampleConfig(1.0, 0.3, True, seed), 1)
        assert len(np.unique(rep.s_h)) < len(rep.s_h)  # duplicates exercised
        assert rel_err(rep.hess_vec(x, v), c["orc_rep_hv"]) <= TOL, i


def test_sparse_newton_trace(sparse_golden):
    for i, A, C, c in sparse_cases(sparse_golden):
        if "records" not in c:
            continue
        ds = CsrDataset.from_scipy(A, c["y"], C)
        cfg = snx.make_variant("subsampled-100", snx.NewtonConfig(max_outer_iters=6))
        tr = snx.newton_solve(snx.SoftmaxProblem(ds, 1e-3), cfg)
        got = np.array([[r.iteration, r.objective, r.train_acc, r.step_size, r.cg_iters]
                        for r in tr.records])
        ref = c["records"]
        assert got.shape == ref.shape
        assert np.array_equal(got[:, [0, 3, 4]], ref[:, [0, 3, 4]]), i
        assert np.allclose(got[:, 1], ref[:, 1], rtol=TOL, atol=0), i
        assert np.array_equal(got[:, 2], ref[:, 2]), i
        assert rel_err(tr.x_final, c["x_final"]) <= 1e-8, i
        tr2 = snx.newton_solve(snx.SoftmaxProblem(ds, 1e-3), cfg)
        assert np.array_equal(tr.x_final, tr2.x_final)  # bit-identical reruns


def test_sparse_matches_dense_path():
    rng = np.random.default_rng(5)
    A = sp.random(3000, 700, density=0.03, format="csr", random_state=5,
                  data_rvs=lambda k: rng.standard_normal(k))
    y = rng.integers(0, 10, 3000)
    x = 0.2 * rng.standard_normal(9 * 700)
    sd = CsrDataset.from_scipy(A, y, 10)
    dd = snx.DeviceDataset.from_numpy(A.toarray(), y, 10)
    ps, pd = snx.SoftmaxProblem(sd, 1e-3), snx.SoftmaxProblem(dd, 1e-3)
    assert abs(snx.objective(ps, x) - snx.objective(pd, x)) <= 1e-12 * abs(snx.objective(pd, x))
    assert rel_err(snx.gradient(ps, x), snx.gradient(pd, x)) <= 1e-12
    # estimate_lipschitz and a CG solve through the sparse operator
    Ls, Ld = snx.estimate_lipschitz(ps, iters=30), snx.estimate_lipschitz(pd, iters=30)
    assert abs(Ls - Ld) <= 1e-10 * Ld
    orc = snx.SubsampledOracle(ps, snx.SampleConfig(1.0, 0.05), 0)
    g = orc.gradient(x)
    rep = snx.cg_solve(orc.hessian_operator(x), g, snx.CgConfig())
    D = A.toarray()
    h = oracle.hess_probs(D[orc.s_h], y[orc.s_h], 10, x)
    sol, _, it, _ = oracle.cg(lambda s: oracle.hess_apply(D[orc.s_h], h, 10, s,
                                                          3000 / len(orc.s_h), 1e-3), g)
    assert rep.iterations == it and rel_err(rep.solution, sol) <= 1e-8


def test_sparse_reference_object_duck_typed():
    """as_device on a reference-style LabeledDataset with CSR features uploads CSR."""
    rng = np.random.default_rng(6)
    A = sp.random(200, 50, density=0.1, format="csr", random_state=6)

    class Feats:
        is_sparse = True
        _mat = sp.csr_array(A)

    class Ds:
        features = Feats()
        labels = rng.integers(0, 4, 200)
        n_classes = 4

    ds = Ds()
    x = 0.1 * rng.standard_normal(3 * 50)
    f = snx.objective(snx.SoftmaxProblem(ds, 0.0), x)
    assert isinstance(snx.as_device(ds), CsrDataset)
    assert abs(f - oracle.loss(A.toarray(), ds.labels, 4, x, 0.0)) <= 1e-12 * abs(f)


def test_load_libsvm_to_device(libsvm_golden):
    """load_libsvm straight to HBM: CSR or dense as the reference picks, and the
    objective / gradient on it equal the oracle's on the reference's parse."""
    from conftest import libsvm_cases

    for name, path, C, nf, storage, g in libsvm_cases(libsvm_golden):
        if str(g["error"]) or not np.all(np.isfinite(g["X"])):
            continue  # parse errors / inf-nan tokens: covered by tests/test_io_cpu.py
        ds = snx.load_libsvm(path, C, n_features=nf, storage=storage)
        assert getattr(ds, "is_sparse", False) == bool(g["is_sparse"]), name
        X, y = g["X"], g["y"]
        x = 0.1 * np.random.default_rng(1).standard_normal((C - 1) * X.shape[1])
        prob = snx.SoftmaxProblem(ds, 1e-3)
        ref = oracle.loss(X, y, C, x, 1e-3)
        assert abs(snx.objective(prob, x) - ref) <= 1e-10 * abs(ref), name
        assert rel_err(snx.gradient(prob, x), oracle.grad(X, y, C, x, 1e-3)) <= 1e-10, name


def test_normalize_columns_csr():
    """normalize_columns on CSR storage (dataset.py:103-118, 314-324): stored
    values of both copies scaled, an empty column untouched."""
    rng = np.random.default_rng(12)
    A = sp.random(700, 90, density=0.05, format="csr", random_state=12,
                  data_rvs=lambda k: rng.standard_normal(k) * 7.0)
    A = A.tolil()
    A[:, 3] = 0.0  # an empty column
    A = sp.csr_array(A.tocsr())
    A.eliminate_zeros()
    y = rng.integers(0, 6, 700)
    ds = CsrDataset.from_scipy(A, y, 6)
    norms, _ = snx.column_norms(ds)
    D = A.toarray()
    assert rel_err(norms.cpu().numpy(), oracle.column_norms(D)) <= 1e-15
    nd = snx.normalize_columns(ds)
    assert isinstance(nd, CsrDataset)
    Dn = oracle.normalize_columns(D)
    got = sp.csr_array((nd.data.cpu().numpy(), nd.indices.cpu().numpy(), nd.indptr.cpu().numpy()),
                       shape=(700, 90)).toarray()
    assert rel_err(got, Dn) <= 1e-15
    x = 0.2 * rng.standard_normal(5 * 90)
    prob = snx.SoftmaxProblem(nd, 1e-3)
    assert rel_err(snx.gradient(prob, x), oracle.grad(Dn, y, 6, x, 1e-3)) <= 1e-10  # CSC copy too


def test_trust_region_and_split_on_csr():
    rng = np.random.default_rng(14)
    A = sp.random(1200, 80, density=0.08, format="csr", random_state=14,
                  data_rvs=lambda k: rng.standard_normal(k))
    y = rng.integers(0, 4, 1200)
    ds = CsrDataset.from_scipy(A, y, 4)
    tr, te = snx.train_test_split(ds, 0.75, 3)
    tri, tei = oracle.train_test_split(1200, 0.75, 3)
    x = 0.1 * rng.standard_normal(3 * 80)
    D = A.toarray()
    assert abs(snx.objective(snx.SoftmaxProblem(tr, 0.0), x) -
               oracle.loss(D[tri], y[tri], 4, x, 0.0)) <= 1e-10 * abs(oracle.loss(D[tri], y[tri], 4, x, 0.0))
    sub_tr, _ = snx.train_test_split(tr, 0.5, 1)  # a split of a view composes the selections
    a, _ = oracle.train_test_split(len(tri), 0.5, 1)
    assert abs(snx.objective(snx.SoftmaxProblem(sub_tr, 0.0), x) -
               oracle.loss(D[tri[a]], y[tri[a]], 4, x, 0.0)) <= 1e-10 * abs(
                   oracle.loss(D[tri[a]], y[tri[a]], 4, x, 0.0))
    cfg = oracle.TrustRegionConfig(max_outer_iters=6)
    ref = oracle.trust_region_solve(D, y, 4, 1e-3, cfg, hessian_fraction=0.1)
    got = snx.trust_region_solve(snx.SoftmaxProblem(ds, 1e-3),
                                 snx.TrustRegionConfig(max_outer_iters=6))
    assert len(got.records) == len(ref["records"])
    for r, (k, f, acc, _, step, it, rad) in zip(got.records, ref["records"]):
        assert r.iteration == k and r.cg_iters == it
        assert abs(r.objective - f) <= 1e-9 * abs(f)
