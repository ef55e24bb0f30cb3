"""Row-sharded path on one GPU: world size 1 must reproduce the unsharded
solver bit for bit, and per-shard partials computed by the CUDA kernels on
shard-local samples must sum to the full-data quantities (the all-reduce
itself is exercised by tests/test_distributed_gloo.py)."""

import numpy as np
import pytest
import torch

import oracle
import paper_1802_09113_b200 as snx
from paper_1802_09113_b200 import distributed as sd
from paper_1802_09113_b200 import softmax
from conftest import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_world1_sharded_newton_matches_unsharded():
    # same kernels; only the CG curvature dot is reduced in a different fixed
    # order (snx_finish_hv's 256 blocks vs the GEMM2 tile partials)
    A, y = oracle.synthetic_problem(3000, 40, 7, seed=21)
    cfg = snx.make_variant("subsampled-20", snx.NewtonConfig(max_outer_iters=5))
    ds = snx.DeviceDataset.from_numpy(A, y, 7)
    ref = snx.newton_solve(snx.SoftmaxProblem(ds, 1e-3), cfg)
    sp = sd.ShardedProblem.from_global(A, y, 7, 1e-3)
    got = sd.newton_solve_sharded(sp, cfg)
    assert got.reason == ref.reason
    assert rel_err(got.x_final, ref.x_final) <= 1e-12
    for a, b in zip(got.records, ref.records):
        assert abs(a.objective - b.objective) <= 1e-13 * abs(b.objective)
        assert a.cg_iters == b.cg_iters and a.step_size == b.step_size
    got2 = sd.newton_solve_sharded(sp, cfg)
    assert np.array_equal(got2.x_final, got.x_final)  # deterministic


def test_two_shards_sum_to_full():
    n, p, C, lam = 4001, 64, 10, 1e-3
    A, y = oracle.synthetic_problem(n, p, C, seed=22)
    x = 0.1 * np.random.default_rng(3).standard_normal((C - 1) * p)
    v = np.random.default_rng(4).standard_normal((C - 1) * p)
    cfg = snx.SampleConfig(1.0, 0.05, seed=3)
    s_g, s_h = snx.draw_samples(cfg, n, 2)
    w = torch.from_numpy(x).cuda()
    vv = torch.from_numpy(v).cuda()
    g_sum = torch.zeros_like(w)
    hv_sum = torch.zeros_like(w)
    loss_sum = 0.0
    for rank in range(2):
        lo, hi = sd.shard_bounds(n, 2, rank)
        sp = sd.ShardedProblem(snx.DeviceDataset.from_numpy(A[lo:hi], y[lo:hi], C), n, lo, lam)
        orc = sd.ShardedOracle(sp, cfg, 2)  # world 1: all_reduce_ is the identity
        g_loc, _ = softmax.gradient_parts(orc._view_g, w, orc.scale_g, 0.0)
        g_sum += g_loc
        op = softmax.HessianOperator(orc._view_h, w, 0.0, scale=orc.scale_h)
        hv_sum += op.apply(vv)
        loss_sum += float(softmax.objective_parts(sp.local, w)[0][0])
    g = g_sum.cpu().numpy() + lam * x
    hv = hv_sum.cpu().numpy() + lam * v
    assert rel_err(g, oracle.grad(A, y, C, x, lam)) <= 1e-10
    h = oracle.hess_probs(A[s_h], y[s_h], C, x)
    assert rel_err(hv, oracle.hess_apply(A[s_h], h, C, v, n / len(s_h), lam)) <= 1e-10
    assert abs(loss_sum - oracle.data_loss(A, y, C, x)) <= 1e-10 * abs(loss_sum)


def test_world1_sharded_full_gradient_pipeline():
    """subsampled-100 (full S_g): the fused trial/gradient pass is reused."""
    A, y = oracle.synthetic_problem(3000, 48, 10, seed=23)
    cfg = snx.make_variant("subsampled-100", snx.NewtonConfig(max_outer_iters=6))
    ds = snx.DeviceDataset.from_numpy(A, y, 10)
    ref = snx.newton_solve(snx.SoftmaxProblem(ds, 1e-3), cfg)
    got = sd.newton_solve_sharded(sd.ShardedProblem.from_global(A, y, 10, 1e-3), cfg)
    assert got.reason == ref.reason
    assert rel_err(got.x_final, ref.x_final) <= 1e-12
    for a, b in zip(got.records, ref.records):
        assert abs(a.objective - b.objective) <= 1e-13 * abs(b.objective)
        assert a.cg_iters == b.cg_iters and a.step_size == b.step_size
        assert a.train_acc == b.train_acc
