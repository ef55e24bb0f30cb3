"""Tensor-core Hessian operator for wide class counts (16 < K <= 128, the
C = 100 configuration of BASELINE.json): h (the wide GEMM1 with the softmax
epilogue) and H v against the fp64 oracle, ragged shapes, reruns bitwise."""

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
