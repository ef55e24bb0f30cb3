"""fp64 data with many classes (C = 18..129, and C = 300 on the loop variant;
csrc/snx_wide64.cu: library DGEMMs + one warp per row) against the CPU oracle
-- the reference computes in fp64 for any C (softmax.py:85-247), so these are fp64 bars: objective / gradient /
h / Hv / probabilities 1e-10 relative, predictions and accuracy exact, CG
iteration counts exact, Newton trajectories as in test_scale_parity_gpu.
Chunking of the logits (zrows < n) is exercised by shrinking the chunk."""

import numpy as np
import pytest
import torch

import oracle
import paper_1802_09113_b200 as snx
from paper_1802_09113_b200 import softmax
from conftest import rel_err

pytestmark = pytest.mark.gpu

SHAPES = [(600, 50, 20), (500, 37, 41), (300, 64, 129), (200, 40, 300)]


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(params=[None, 128], ids=["one-chunk", "chunked"])
def zrows(request, monkeypatch):
    if request.param is not None:
        monkeypatch.setattr(softmax, "_ZROWS", request.param)
    return request.param


@pytest.mark.parametrize("n,p,C", SHAPES)
def test_objective_gradient_probabilities(n, p, C, zrows):
    A, y = oracle.synthetic_problem(n, p, C, seed=C)
    x = 0.3 * np.random.default_rng(p).standard_normal((C - 1) * p)
    lam = 1e-3
    ds = snx.DeviceDataset.from_numpy(A, y, C)
    prob = snx.SoftmaxProblem(ds, lam)
    f = snx.objective(prob, x)
    f_ref = oracle.loss(A, y, C, x, lam)
    assert abs(f - f_ref) <= 1e-10 * abs(f_ref)
    g = snx.gradient(prob, x)
    assert rel_err(g, oracle.grad(A, y, C, x, lam)) <= 1e-10
    assert np.array_equal(snx.gradient(prob, x), g)  # rerun bit-identical
    assert snx.accuracy(ds, x) == oracle.accuracy(A, y, C, x)
    P = snx.class_probabilities(ds, x)
    assert P.shape == (n, C)
    assert rel_err(P, oracle.class_probs(A, y, C, x)) <= 1e-12
    assert np.array_equal(snx.predict(ds, x), oracle.predict(A, y, C, x))
    M, E, alpha, lin = oracle.row_terms(A, y, oracle.weights_matrix(x, p, C), C)
    rs = snx.row_stats(ds, x)
    assert rel_err(rs.max_part, M) <= 1e-12
    assert rel_err(rs.sum_exp_part, E.sum(axis=1)) <= 1e-12
    assert rel_err(rs.linear_part, lin) <= 1e-12


@pytest.mark.parametrize("n,p,C", SHAPES)
def test_hessian_and_cg(n, p, C, zrows):
    A, y = oracle.synthetic_problem(n, p, C, seed=2 * C)
    rng = np.random.default_rng(C)
    x = 0.2 * rng.standard_normal((C - 1) * p)
    v = rng.standard_normal((C - 1) * p)
    lam = 1e-2
    ds = snx.DeviceDataset.from_numpy(A, y, C)
    orc = snx.SubsampledOracle(snx.SoftmaxProblem(ds, lam), snx.SampleConfig(1.0, 0.4), 3)
    s_h = orc.s_h
    op = orc.hessian_operator(x)
    h = oracle.hess_probs(A[s_h], y[s_h], C, x)
    assert rel_err(op._h.cpu().numpy(), h) <= 1e-12
    scale = n / len(s_h)
    hv = op.apply(v)
    assert rel_err(hv, oracle.hess_apply(A[s_h], h, C, v, scale, lam)) <= 1e-10
    assert np.array_equal(op.apply(v), hv)
    g = oracle.grad(A, y, C, x, lam)
    rep = snx.cg_solve(op, g, snx.CgConfig(1e-6, 8))
    p_ref, rn_ref, it_ref, conv_ref = oracle.cg(
        lambda u: oracle.hess_apply(A[s_h], h, C, u, scale, lam), g, 1e-6, 8)
    assert rep.iterations == it_ref and rep.converged == conv_ref
    assert rel_err(rep.solution, p_ref) <= 1e-9


def test_newton_trajectory_wide_classes():
    """subsampled-20 Newton at C = 40 (fresh samples every iteration, the device
    CG on the wide product, Armijo on the wide objective) = the oracle's."""
    n, p, C, lam = 2000, 96, 40, 1e-3
    A, y = oracle.synthetic_problem(n, p, C, seed=11)
    ref = oracle.newton_solve(A, y, C, lam, "subsampled-20", max_outer_iters=4)
    ds = snx.DeviceDataset.from_numpy(A, y, C)
    tr = snx.newton_solve(snx.SoftmaxProblem(ds, lam),
                          snx.make_variant("subsampled-20", snx.NewtonConfig(max_outer_iters=4)))
    recs = ref["records"]
    assert tr.reason == ref["reason"] and len(tr.records) == len(recs)
    for r, (k, f, acc, _, alpha, it) in zip(tr.records, recs):
        assert abs(r.objective - f) <= 1e-10 * abs(f), (k, r.objective, f)
        assert r.step_size == alpha and r.cg_iters == it, k
        assert r.train_acc == acc, k
    assert rel_err(tr.x_final, ref["x"]) <= 1e-9


def test_f32_wide_probabilities():
    """f32 data with C = 60: class_probabilities / predict / row_stats widen each
    row chunk to fp64 (the fp64 path on the f32-rounded data): 1e-12 against the
    oracle on the rounded data, predictions exact."""
    n, p, C = 700, 45, 60
    A, y = oracle.synthetic_problem(n, p, C, seed=4)
    A32 = A.astype(np.float32).astype(np.float64)
    x = 0.3 * np.random.default_rng(5).standard_normal((C - 1) * p)
    ds = snx.DeviceDataset.from_numpy(A, y, C, dtype="f32")
    P = snx.class_probabilities(ds, x)
    assert rel_err(P, oracle.class_probs(A32, y, C, x)) <= 1e-12
    assert np.array_equal(snx.predict(ds, x), oracle.predict(A32, y, C, x))
    M, E, alpha, lin = oracle.row_terms(A32, y, oracle.weights_matrix(x, p, C), C)
    rs = snx.row_stats(ds, x)
    assert rel_err(rs.sum_exp_part, E.sum(axis=1)) <= 1e-12
    assert rel_err(rs.linear_part, lin) <= 1e-12


@pytest.mark.parametrize("C", [40, 150])
def test_csr_wide_classes(C):
    """CSR storage with C > 33 (the wide row kernels behind a warp-per-row CSR
    logits pass and a warp-per-column CSC X^T R pass): objective, gradient,
    accuracy, probabilities, the sampled product (with duplicate rows), CG and
    a short Newton trajectory against the oracle on the dense matrix."""
    import scipy.sparse as sp

    from paper_1802_09113_b200.sparse import CsrDataset

    n, p, lam = 900, 120, 1e-3
    rng = np.random.default_rng(C)
    As = sp.random(n, p, density=0.08, format="csr", random_state=C)
    A = As.toarray()
    y = rng.integers(0, C, size=n)
    x = 0.3 * rng.standard_normal((C - 1) * p)
    v = rng.standard_normal((C - 1) * p)
    ds = CsrDataset.from_scipy(As, y, C)
    prob = snx.SoftmaxProblem(ds, lam)
    f_ref = oracle.loss(A, y, C, x, lam)
    assert abs(snx.objective(prob, x) - f_ref) <= 1e-10 * abs(f_ref)
    assert rel_err(snx.gradient(prob, x), oracle.grad(A, y, C, x, lam)) <= 1e-10
    assert snx.accuracy(ds, x) == oracle.accuracy(A, y, C, x)
    assert rel_err(snx.class_probabilities(ds, x), oracle.class_probs(A, y, C, x)) <= 1e-12
    orc = snx.SubsampledOracle(prob, snx.SampleConfig(1.0, 0.3, True, 7), 1)
    s_h = orc.s_h
    assert len(np.unique(s_h)) < len(s_h)  # duplicates
    h = oracle.hess_probs(A[s_h], y[s_h], C, x)
    scale = n / len(s_h)
    op = orc.hessian_operator(x)
    assert rel_err(op.apply(v), oracle.hess_apply(A[s_h], h, C, v, scale, lam)) <= 1e-10
    g = oracle.grad(A, y, C, x, lam)
    rep = snx.cg_solve(op, g, snx.CgConfig(1e-6, 6))
    p_ref, _, it_ref, conv_ref = oracle.cg(
        lambda u: oracle.hess_apply(A[s_h], h, C, u, scale, lam), g, 1e-6, 6)
    assert rep.iterations == it_ref and rep.converged == conv_ref
    assert rel_err(rep.solution, p_ref) <= 1e-9
    ref = oracle.newton_solve(A, y, C, lam, "subsampled-100", max_outer_iters=3)
    tr = snx.newton_solve(prob, snx.make_variant("subsampled-100",
                                                 snx.NewtonConfig(max_outer_iters=3)))
    for r, (k, f, acc, _, alpha, it) in zip(tr.records, ref["records"]):
        assert abs(r.objective - f) <= 1e-10 * abs(f), k
        assert r.step_size == alpha and r.cg_iters == it, k
    assert rel_err(tr.x_final, ref["x"]) <= 1e-9
