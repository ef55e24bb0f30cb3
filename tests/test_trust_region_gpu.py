"""Device-resident Steihaug-CG (BASELINE config #4) against the CPU
restatement oracle/trust_region.py (parity unpinned against the reference,
which has no trust-region solver): every branch -- interior convergence,
iteration cap, boundary hit, zero gradient."""

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


@pytest.mark.parametrize("radius,theta,T", [(1e3, 1e-4, 10), (1e3, 1e-12, 4), (0.05, 1e-4, 10),
                                            (1e-6, 1e-4, 10), (2.0, 1e-3, 25)])
def test_steihaug_branches(radius, theta, T):
    A, y = oracle.synthetic_problem(3000, 40, 6, seed=11)
    x = 0.2 * np.random.default_rng(3).standard_normal(5 * 40)
    g = oracle.grad(A, y, 6, x, 1e-3)
    h = oracle.hess_probs(A, y, 6, x)
    ref = oracle.steihaug_cg(lambda v: oracle.hess_apply(A, h, 6, v, 1.0, 1e-3), g, radius,
                             theta, T)
    ds = snx.DeviceDataset.from_numpy(A, y, 6)
    op = snx.HessianOperator(ds, x, 1e-3)
    gd = torch.from_numpy(g).cuda()
    p, m, it, bnd = snx.steihaug_cg(op, gd, radius, theta, T)
    assert it == ref[2] and bnd == ref[3], (it, ref[2], bnd, ref[3])
    assert rel_err(p.cpu().numpy(), ref[0]) <= 1e-9
    assert abs(m - ref[1]) <= 1e-9 * abs(ref[1])
    if bnd:
        assert abs(float(torch.linalg.vector_norm(p)) - radius) <= 1e-9 * radius


def test_steihaug_zero_gradient():
    A, y = oracle.synthetic_problem(200, 8, 3, seed=2)
    ds = snx.DeviceDataset.from_numpy(A, y, 3)
    op = snx.HessianOperator(ds, np.zeros(16), 1e-3)
    p, m, it, bnd = snx.steihaug_cg(op, torch.zeros(16, dtype=torch.float64, device="cuda"),
                                    1.0, 1e-4, 10)
    assert it == 0 and m == 0.0 and not bnd and float(p.abs().sum()) == 0.0


def test_trust_region_cifar_shape_matches_restatement():
    A, y = oracle.synthetic_problem(5000, 512, 10, seed=0, normalize=False,
                                    ill_conditioned=True)
    cfg = oracle.TrustRegionConfig(max_outer_iters=8)
    ref = oracle.trust_region_solve(A, y, 10, 1e-3, cfg, hessian_fraction=0.1)
    ds = snx.DeviceDataset.from_numpy(A, y, 10)
    tr = snx.trust_region_solve(snx.SoftmaxProblem(ds, 1e-3),
                                snx.TrustRegionConfig(max_outer_iters=8))
    assert len(tr.records) == len(ref["records"])
    for r, (k, f, acc, _, step, it, rad) in zip(tr.records, ref["records"]):
        assert r.iteration == k and r.cg_iters == it
        assert abs(r.objective - f) <= 1e-9 * abs(f)
        assert abs(r.step_size - step) <= 1e-7 * max(1.0, step)
    assert tr.reason == ref["reason"]
