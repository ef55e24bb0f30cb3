"""Solver edge cases against the oracle (pinned to the reference by
tests/test_oracle_golden.py): sampling with replacement (duplicate rows in
S_g / S_H, sampling.py:41-42), the subsampled-20 variant's small gradient
sample, a warm start at the optimum (tests/test_newton.py:77-85), two-class
(logistic) and 17-class (K = 16, the largest fp64 template) problems."""

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


def _trace(tr):
    return np.array([[r.iteration, r.objective, r.train_acc, r.step_size, r.cg_iters]
                     for r in tr.records])


def _ref_trace(ref):
    return np.array([[r[0], r[1], r[2], r[4], r[5]] for r in ref["records"]])


@pytest.mark.parametrize("n,p,C,fg,fh,repl", [(1500, 30, 5, 1.0, 0.3, True),
                                               (2000, 24, 4, 0.2, 0.05, True),
                                               (900, 16, 2, 1.0, 0.1, False),
                                               (1200, 20, 17, 0.5, 0.2, False)])
def test_newton_variants_vs_oracle(n, p, C, fg, fh, repl):
    A, y = oracle.synthetic_problem(n, p, C, seed=n + C)
    cfg = snx.NewtonConfig(max_outer_iters=6,
                           samples=snx.SampleConfig(fg, fh, repl, seed=5))
    tr = snx.newton_solve(snx.SoftmaxProblem(snx.DeviceDataset.from_numpy(A, y, C), 1e-3), cfg)
    ref = oracle.newton_solve(A, y, C, 1e-3, seed=5, max_outer_iters=6, with_replacement=repl,
                              gradient_fraction=fg, hessian_fraction=fh)
    got, exp = _trace(tr), _ref_trace(ref)
    assert got.shape == exp.shape and tr.reason == ref["reason"]
    assert np.array_equal(got[:, [0, 3, 4]], exp[:, [0, 3, 4]])
    assert np.allclose(got[:, 1], exp[:, 1], rtol=1e-10, atol=0)
    assert np.array_equal(got[:, 2], exp[:, 2])
    assert rel_err(tr.x_final, ref["x"]) <= 1e-8


def test_warm_start_at_optimum_converges_immediately():
    A, y = oracle.synthetic_problem(800, 12, 3, seed=4)
    ds = snx.DeviceDataset.from_numpy(A, y, 3)
    prob = snx.SoftmaxProblem(ds, 1e-2)
    full = snx.make_variant("full", snx.NewtonConfig(max_outer_iters=30, epsilon=1e-9))
    tr = snx.newton_solve(prob, full)
    assert tr.reason == "gradient-converged"
    again = snx.newton_solve(prob, full, x0=tr.x_final)
    assert again.reason == "gradient-converged" and again.iterations == 0
    assert np.array_equal(again.x_final, tr.x_final)


def test_sampled_oracle_with_replacement_dense():
    A, y = oracle.synthetic_problem(3000, 40, 6, seed=9)
    x = 0.2 * np.random.default_rng(1).standard_normal(5 * 40)
    v = np.random.default_rng(2).standard_normal(5 * 40)
    cfg = snx.SampleConfig(0.4, 0.3, True, seed=2)
    orc = snx.SubsampledOracle(snx.SoftmaxProblem(snx.DeviceDataset.from_numpy(A, y, 6), 1e-3),
                               cfg, 3)
    s_g, s_h = oracle.draw_samples(0.4, 0.3, True, 2, 3000, 3)
    assert np.array_equal(orc.s_g, s_g) and np.array_equal(orc.s_h, s_h)
    assert len(np.unique(s_h)) < len(s_h)
    g_ref = oracle.grad(A[s_g], y[s_g], 6, x, 1e-3, scale=3000 / len(s_g))
    assert rel_err(orc.gradient(x), g_ref) <= 1e-10
    h = oracle.hess_probs(A[s_h], y[s_h], 6, x)
    hv_ref = oracle.hess_apply(A[s_h], h, 6, v, 3000 / len(s_h), 1e-3)
    assert rel_err(orc.hess_vec(x, v), hv_ref) <= 1e-10
