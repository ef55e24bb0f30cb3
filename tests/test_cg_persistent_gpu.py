"""The persistent one-launch CG solve (snx_cg_solve) against the per-iteration
path (snx_hess_apply + snx_cg_update): bit-identical CG state, on ragged
shapes, early convergence, a zero right-hand side and whole Newton solves."""

import numpy as np
import pytest
import torch

import oracle
import paper_1802_09113_b200 as snx
from paper_1802_09113_b200 import cg as cgmod, softmax

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _solve(op, g, theta, T, persistent, monkeypatch):
    # the persistent solve replicates the unfused per-iteration path
    monkeypatch.setenv("SNX_CG_FUSED", "0")
    monkeypatch.setenv("SNX_CG_PERSISTENT", "1" if persistent else "0")
    ws = cgmod.CgWorkspace(op.dim, T, g.device)
    cgmod.enqueue_cg(op, g, theta, T, ws)
    torch.cuda.synchronize()
    return ws


@pytest.mark.parametrize("n,p,C,frac,theta,T", [
    (3001, 130, 5, 0.3, 1e-4, 10), (6000, 300, 10, 0.05, 1e-4, 10), (129, 33, 17, 1.0, 1e-6, 12),
    (1, 7, 3, 1.0, 1e-4, 4), (5000, 200, 10, 0.1, 0.5, 10), (2500, 3072, 10, 1.0, 1e-4, 10)])
def test_persistent_cg_bit_identical(n, p, C, frac, theta, T, monkeypatch):
    A, y = oracle.synthetic_problem(n, p, C, seed=n)
    ds = snx.DeviceDataset.from_numpy(A, y, C)
    x = torch.from_numpy(0.1 * np.random.default_rng(1).standard_normal((C - 1) * p)).cuda()
    view = ds.take(snx.draw_samples(snx.SampleConfig(1.0, frac), n, 0)[1])
    op = softmax.HessianOperator(view, x, 1e-3, scale=n / view.n_rows)
    g, _ = softmax.gradient_parts(ds, x, 1.0, 1e-3)
    ref = _solve(op, g, theta, T, False, monkeypatch)
    got = _solve(op, g, theta, T, True, monkeypatch)
    assert torch.equal(got.state[:(T + 1) * 8], ref.state[:(T + 1) * 8])
    for name in ("pb", "r", "s", "p", "Hs"):
        assert torch.equal(getattr(got, name), getattr(ref, name)), name
    rep = cgmod.report_from(got, T, True)
    assert rep.iterations == cgmod.report_from(ref, T, True).iterations


def test_persistent_cg_zero_rhs(monkeypatch):
    A, y = oracle.synthetic_problem(500, 20, 4, seed=2)
    ds = snx.DeviceDataset.from_numpy(A, y, 4)
    x = torch.zeros(60, dtype=torch.float64, device="cuda")
    op = softmax.HessianOperator(ds, x, 1e-3)
    g = torch.zeros(60, dtype=torch.float64, device="cuda")
    ws = _solve(op, g, 1e-4, 5, True, monkeypatch)
    rep = cgmod.report_from(ws, 5, True)
    assert rep.iterations == 0 and rep.converged and float(rep.solution.abs().sum()) == 0.0


def test_persistent_newton_trace_identical(monkeypatch):
    A, y = oracle.synthetic_problem(4000, 60, 10, seed=9)
    cfg = snx.make_variant("subsampled-20", snx.NewtonConfig(max_outer_iters=6))
    ds = snx.DeviceDataset.from_numpy(A, y, 10)
    monkeypatch.setenv("SNX_CG_FUSED", "0")
    monkeypatch.setenv("SNX_CG_PERSISTENT", "0")
    ref = snx.newton_solve(snx.SoftmaxProblem(ds, 1e-3), cfg)
    monkeypatch.setenv("SNX_CG_PERSISTENT", "1")
    got = snx.newton_solve(snx.SoftmaxProblem(ds, 1e-3), cfg)
    assert np.array_equal(got.x_final, ref.x_final)
    assert [r.cg_iters for r in got.records] == [r.cg_iters for r in ref.records]


@pytest.mark.parametrize("n,p,C,frac,theta,T", [
    (3001, 130, 5, 0.3, 1e-4, 10), (6000, 300, 10, 0.05, 1e-4, 10), (129, 33, 17, 1.0, 1e-6, 12),
    (1, 7, 3, 1.0, 1e-4, 4), (5000, 200, 10, 0.1, 0.5, 10), (2500, 3072, 10, 1.0, 1e-4, 10),
    (40000, 784, 10, 0.05, 1e-4, 10)])
def test_fused_cg_matches_unfused(n, p, C, frac, theta, T, monkeypatch):
    """snx_hess_apply_cg (CG update in GEMM2's tail) vs apply + snx_cg_update:
    same iteration counts and flags, iterates equal to rounding (the r.r sum
    is ordered by column tiles instead of 256 blocks); fused reruns bitwise."""
    A, y = oracle.synthetic_problem(n, p, C, seed=n)
    ds = snx.DeviceDataset.from_numpy(A, y, C)
    x = torch.from_numpy(0.1 * np.random.default_rng(1).standard_normal((C - 1) * p)).cuda()
    view = ds.take(snx.draw_samples(snx.SampleConfig(1.0, frac), n, 0)[1])
    op = softmax.HessianOperator(view, x, 1e-3, scale=n / view.n_rows)
    g, _ = softmax.gradient_parts(ds, x, 1.0, 1e-3)

    def run(fused):
        monkeypatch.setenv("SNX_CG_PERSISTENT", "0")
        monkeypatch.setenv("SNX_CG_FUSED", "1" if fused else "0")
        ws = cgmod.CgWorkspace(op.dim, T, g.device)
        cgmod.enqueue_cg(op, g, theta, T, ws)
        torch.cuda.synchronize()
        return ws

    ref, got, again = run(False), run(True), run(True)
    a, b = cgmod.report_from(got, T, True), cgmod.report_from(ref, T, True)
    assert (a.iterations, a.converged) == (b.iterations, b.converged)
    st_g, st_r = got.state[:(T + 1) * 8].view(T + 1, 8), ref.state[:(T + 1) * 8].view(T + 1, 8)
    assert torch.equal(st_g[:, [2, 3, 4, 6]], st_r[:, [2, 3, 4, 6]])  # done, iters, conv, err
    assert torch.allclose(st_g[:, [0, 1, 5]], st_r[:, [0, 1, 5]], rtol=1e-12, atol=0)
    sol, sol_ref = a.solution, b.solution
    assert float((sol - sol_ref).norm() / sol_ref.norm()) <= 1e-11
    assert torch.equal(again.pb, got.pb) and torch.equal(again.state, got.state)
