"""The one-pass row pass (csrc/snx_cluster.cu) over every plan it picks, against
the CPU oracle (the reference's arithmetic):

  * column split with 1-, 2-, 4- and 8-CTA clusters (p = 200, 900, 2000, 5000:
    slices of 200 .. 626 columns, ragged against the 16-column chunks and the
    16-column X^T U tiles), and the row split (p = 40);
  * K = 1, 4 and 9 free classes (class 8 on the DFMA side path);
  * the three modes: prep (h), apply (Hv, and the fused CG iteration), grad
    (full-data gradient + loss + accuracy, two row-algebra warps);
  * sample sizes with one block per cluster, odd block counts, a single row.

Bars: h 1e-12, Hv / gradient / objective 1e-10 relative (fp64), CG iteration
counts exact and the solution 1e-9; reruns bit-identical."""

import numpy as np
import pytest
import torch

import oracle
import paper_1802_09113_b200 as snx
from conftest import rel_err

pytestmark = pytest.mark.gpu

SHAPES = [  # n, p, C: plan
    (2000, 40, 10),     # row split
    (3000, 200, 10),    # 1-CTA clusters
    (3000, 900, 5),     # 2-CTA clusters
    (2500, 2000, 10),   # 4-CTA clusters
    (1200, 5000, 2),    # 8-CTA clusters, K = 1
]


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("n,p,C", SHAPES)
@pytest.mark.parametrize("f_h", [0.05, 0.31])
def test_product_prepare_and_cg(n, p, C, f_h):
    A, y = oracle.synthetic_problem(n, p, C, seed=p + C)
    rng = np.random.default_rng(p)
    x = 0.1 * rng.standard_normal((C - 1) * p)
    v = rng.standard_normal((C - 1) * p)
    lam = 1e-3
    ds = snx.DeviceDataset.from_numpy(A, y, C)
    prob = snx.SoftmaxProblem(ds, lam)
    orc = snx.SubsampledOracle(prob, snx.SampleConfig(1.0, f_h), 3)
    s_h = orc.s_h
    op = orc.hessian_operator(x)
    h_ref = oracle.hess_probs(A[s_h], y[s_h], C, x)
    assert rel_err(op._h.cpu().numpy(), h_ref) <= 1e-12
    scale = n / len(s_h)
    hv_ref = oracle.hess_apply(A[s_h], h_ref, C, v, scale, lam)
    hv = op.apply(v)
    assert rel_err(hv, hv_ref) <= 1e-10
    assert np.array_equal(op.apply(v), hv)  # rerun bit-identical
    # the CG solve on the fused path (product + finalize + CG update per iteration)
    g = oracle.grad(A, y, C, x, lam)
    rep = snx.cg_solve(op, g, snx.CgConfig(1e-6, 8))
    p_ref, rn_ref, it_ref, conv_ref = oracle.cg(
        lambda u: oracle.hess_apply(A[s_h], h_ref, C, u, scale, lam), g, 1e-6, 8)
    assert rep.iterations == it_ref and rep.converged == conv_ref
    assert rel_err(rep.solution, p_ref) <= 1e-9
    assert abs(rep.residual_norm - rn_ref) <= 1e-9 * max(rn_ref, 1e-300)


@pytest.mark.parametrize("n,p,C", SHAPES)
def test_full_gradient_objective_accuracy(n, p, C):
    A, y = oracle.synthetic_problem(n, p, C, seed=7 * p + C)
    x = 0.2 * np.random.default_rng(C).standard_normal((C - 1) * p)
    lam = 1e-3
    ds = snx.DeviceDataset.from_numpy(A, y, C)
    prob = snx.SoftmaxProblem(ds, lam)
    g = snx.gradient(prob, x)
    assert rel_err(g, oracle.grad(A, y, C, x, lam)) <= 1e-10
    assert np.array_equal(snx.gradient(prob, x), g)
    f = snx.objective(prob, x)
    f_ref = oracle.loss(A, y, C, x, lam)
    assert abs(f - f_ref) <= 1e-10 * abs(f_ref)
    assert snx.accuracy(prob.dataset, x) == oracle.accuracy(A, y, C, x)


@pytest.mark.parametrize("m", [1, 7, 8, 9, 63, 65])
def test_tiny_samples(m):
    """Fewer sample rows than clusters (empty clusters, a partial last block)."""
    n, p, C = 400, 2000, 10
    A, y = oracle.synthetic_problem(n, p, C, seed=m)
    rng = np.random.default_rng(m)
    x = 0.1 * rng.standard_normal((C - 1) * p)
    v = rng.standard_normal((C - 1) * p)
    rows = np.sort(rng.choice(n, m, replace=False))
    ds = snx.DeviceDataset.from_numpy(A, y, C)
    op = snx.softmax.HessianOperator(ds.take(rows), x, 1e-3, scale=n / m)
    h = oracle.hess_probs(A[rows], y[rows], C, x)
    ref = oracle.hess_apply(A[rows], h, C, v, n / m, 1e-3)
    assert rel_err(op.apply(v), ref) <= 1e-10


@pytest.mark.parametrize("n,p,C", [(2000, 40, 10), (3000, 900, 5), (2500, 2000, 10)])
def test_f32_rows_widened(n, p, C):
    """f32 data on the one-pass kernel (rows copied as f32, widened to fp64 in
    shared memory): the fp64 arithmetic on the f32-rounded data, so the product
    and the gradient match the oracle on the rounded data to 1e-10 and the
    original data to the declared 1e-4."""
    A, y = oracle.synthetic_problem(n, p, C, seed=p)
    A32 = A.astype(np.float32).astype(np.float64)
    rng = np.random.default_rng(C)
    x = 0.1 * rng.standard_normal((C - 1) * p)
    v = rng.standard_normal((C - 1) * p)
    lam = 1e-3
    ds = snx.DeviceDataset.from_numpy(A, y, C, dtype="f32")
    prob = snx.SoftmaxProblem(ds, lam)
    orc = snx.SubsampledOracle(prob, snx.SampleConfig(1.0, 0.2), 1)
    op = orc.hessian_operator(x)
    assert op._bufs.fused and op._bufs.xs_tc is None
    s_h = orc.s_h
    h = oracle.hess_probs(A32[s_h], y[s_h], C, x)
    ref = oracle.hess_apply(A32[s_h], h, C, v, n / len(s_h), lam)
    hv = op.apply(v)
    assert rel_err(hv, ref) <= 1e-10
    assert rel_err(hv, oracle.hess_apply(A[s_h], oracle.hess_probs(A[s_h], y[s_h], C, x), C, v,
                                         n / len(s_h), lam)) <= 1e-4
    assert rel_err(snx.gradient(prob, x), oracle.grad(A32, y, C, x, lam)) <= 1e-10


@pytest.mark.parametrize("n,p,C", SHAPES)
def test_cg_early_stop_skips_products(n, p, C):
    """A loose tolerance stops CG after a few iterations: the remaining products
    of the captured solve see the done flag and leave (the producer completes the
    ring stages it staged before griddepcontrol.wait); the result is the
    oracle's, and a second solve on the same graph reproduces it bit for bit."""
    A, y = oracle.synthetic_problem(n, p, C, seed=3 * p + C)
    rng = np.random.default_rng(n)
    x = 0.1 * rng.standard_normal((C - 1) * p)
    lam = 1e-2
    ds = snx.DeviceDataset.from_numpy(A, y, C)
    orc = snx.SubsampledOracle(snx.SoftmaxProblem(ds, lam), snx.SampleConfig(1.0, 0.2), 5)
    op = orc.hessian_operator(x)
    s_h = orc.s_h
    h = oracle.hess_probs(A[s_h], y[s_h], C, x)
    g = oracle.grad(A, y, C, x, lam)
    scale = n / len(s_h)
    rep = snx.cg_solve(op, g, snx.CgConfig(0.5, 10))
    p_ref, rn_ref, it_ref, conv_ref = oracle.cg(
        lambda u: oracle.hess_apply(A[s_h], h, C, u, scale, lam), g, 0.5, 10)
    assert conv_ref and it_ref < 10
    assert rep.iterations == it_ref and rep.converged
    assert rel_err(rep.solution, p_ref) <= 1e-9
    rep2 = snx.cg_solve(op, g, snx.CgConfig(0.5, 10))
    assert np.array_equal(rep2.solution, rep.solution)
