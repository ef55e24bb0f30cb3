"""Tensor-core Hessian operator for wide class counts (16 < K <= 128, the
C = 100 configuration of BASELINE.json): h (the wide GEMM1 with the softmax
epilogue) and H v against the fp64 oracle, ragged shapes, reruns bitwise."""

import math

import numpy as np
import pytest
import torch

import oracle
import paper_1802_09113_b200 as snx
from conftest import rel_err

pytestmark = pytest.mark.gpu

TOL_TC = 2e-5  # declared f32 bar: 1e-4


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("n,p,C,frac", [(700, 130, 18, 1.0), (2000, 257, 33, 0.5),
                                        (3001, 300, 100, 0.3), (1500, 96, 129, 1.0),
                                        (129, 65, 64, 1.0)])
def test_wide_hessian_vs_oracle(n, p, C, frac):
    A, y = oracle.synthetic_problem(n, p, C, seed=C)
    rng = np.random.default_rng(C)
    x = 0.3 * rng.standard_normal((C - 1) * p)
    v = rng.standard_normal((C - 1) * p)
    prob = snx.SoftmaxProblem(snx.DeviceDataset.from_numpy(A, y, C, dtype="f32"), 1e-3)
    orc = snx.SubsampledOracle(prob, snx.SampleConfig(1.0, frac, seed=2), 1)
    s_h = orc.s_h
    op = orc.hessian_operator(x)
    h_ref = oracle.hess_probs(A[s_h], y[s_h], C, x)
    assert rel_err(op._h.double().cpu().numpy(), h_ref) <= TOL_TC
    ref = oracle.hess_apply(A[s_h], h_ref, C, v, n / len(s_h), 1e-3)
    got = op.apply(v)
    assert rel_err(got, ref) <= TOL_TC, rel_err(got, ref)
    assert np.array_equal(op.apply(v), got)


@pytest.mark.parametrize("n,p,C", [(3001, 130, 18), (2500, 257, 100), (0, 40, 33), (1, 9, 129)])
def test_wide_objective_gradient_vs_oracle(n, p, C):
    A, y = oracle.synthetic_problem(max(n, 1), p, C, seed=C + 1)
    A, y = A[:n], y[:n]
    rng = np.random.default_rng(C)
    x = 0.3 * rng.standard_normal((C - 1) * p)
    d = rng.standard_normal((C - 1) * p)
    ds = snx.DeviceDataset.from_numpy(A, y, C, dtype="f32")
    prob = snx.SoftmaxProblem(ds, 1e-3)
    f = snx.objective(prob, x)
    f_ref = oracle.loss(A, y, C, x, 1e-3)
    assert abs(f - f_ref) <= TOL_TC * max(1.0, abs(f_ref))
    assert rel_err(snx.gradient(prob, x), oracle.grad(A, y, C, x, 1e-3)) <= TOL_TC
    # line-search trial point and accuracy through the same pass
    w = torch.from_numpy(x).cuda()
    out, corr = snx.softmax.objective_parts(ds, w, torch.from_numpy(d).cuda(), 0.25,
                                            want_correct=True)
    xt = x + 0.25 * d
    assert abs(float(out[0]) - oracle.data_loss(A, y, C, xt)) <= TOL_TC * max(
        1.0, abs(oracle.data_loss(A, y, C, xt)))
    assert abs(float(out[1]) - float(xt @ xt)) <= 1e-12 * float(xt @ xt)
    if n:
        acc_ref = oracle.accuracy(A, y, C, xt)
        assert abs(int(corr) / n - acc_ref) <= 2.0 / n


def test_wide_newton_solve_matches_oracle():
    n, p, C = 4000, 60, 40
    A, y = oracle.synthetic_problem(n, p, C, seed=3)
    cfg = snx.make_variant("subsampled-20", snx.NewtonConfig(max_outer_iters=5))
    tr = snx.newton_solve(snx.SoftmaxProblem(snx.DeviceDataset.from_numpy(A, y, C, dtype="f32"),
                                             1e-3), cfg)
    ref = oracle.newton_solve(A, y, C, 1e-3, variant="subsampled-20", max_outer_iters=5)
    ref_f = [r[1] for r in ref["records"]]
    assert len(tr.records) == len(ref_f)
    for a, b in zip(tr.records, ref_f):
        assert abs(a.objective - b) <= 1e-4 * abs(b)


def test_config5_shard_properties_full_size():
    """BASELINE config #5 at its per-GPU size (1M x 3072 f32 rows, C = 100, 5%
    sample): too large for the oracle, so size-independent properties of the
    sampled Hessian: symmetry u.Hv = v.Hu, linearity, positive curvature, and
    bit-identical reruns (fixed-order reductions)."""
    n, p, C = 1_000_000, 3072, 100
    K = C - 1
    g = torch.Generator(device="cuda").manual_seed(5)
    X = torch.randn((n, p), generator=g, device="cuda", dtype=torch.float32) / math.sqrt(n)
    lab = torch.randint(0, C, (n,), generator=g, device="cuda", dtype=torch.int32)
    ds = snx.DeviceDataset(X, lab, C, p, dtype="f32")
    x = 0.05 * torch.randn(K * p, generator=g, device="cuda", dtype=torch.float64)
    u = torch.randn(K * p, generator=g, device="cuda", dtype=torch.float64)
    v = torch.randn(K * p, generator=g, device="cuda", dtype=torch.float64)
    orc = snx.SubsampledOracle(snx.SoftmaxProblem(ds, 1e-3), snx.SampleConfig(1.0, 0.05), 0)
    op = orc.hessian_operator(x)
    Hu, Hv = op.apply(u), op.apply(v)
    uHv, vHu = float(u @ Hv), float(v @ Hu)
    assert abs(uHv - vHu) <= 1e-4 * max(abs(uHv), 1e-30)
    assert float(u @ Hu) > 0 and float(v @ Hv) > 0
    w = 0.3 * u - 2.0 * v
    Hw = op.apply(w)
    lin = 0.3 * Hu - 2.0 * Hv
    assert float(torch.linalg.vector_norm(Hw - lin) / torch.linalg.vector_norm(lin)) <= 1e-4
    assert torch.equal(op.apply(u), Hu)
    del X, ds, op
    torch.cuda.empty_cache()
