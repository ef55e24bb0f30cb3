"""class_probabilities / predict / row_stats (softmax.py:107-122, 224-240) on the
device against the reference's golden values; CSR storage against the oracle."""

import numpy as np
import pytest
import scipy.sparse as sp
import torch

import oracle
import paper_1802_09113_b200 as snx
from conftest import rel_err, softmax_cases
from paper_1802_09113_b200.sparse import CsrDataset

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-10), ("f32", 1e-4)])
def test_probs_predict_rowstats_golden(softmax_golden, dtype, tol):
    seen = 0
    for i, c in softmax_cases(softmax_golden):
        n, p, C = (int(t) for t in c["shape"])
        if n == 0 or (dtype == "f32" and i == 3):
            continue
        ds = snx.DeviceDataset.from_numpy(c["A"], c["y"], C, dtype=dtype)
        x = c["x"]
        P = snx.class_probabilities(ds, x)
        assert P.shape == (n, C)
        assert rel_err(P, c["probs"]) <= tol, i
        rs = snx.row_stats(ds, x)
        assert rel_err(rs.max_part, c["row_max"]) <= tol, i
        assert rel_err(rs.sum_exp_part, c["row_sumexp"]) <= tol, i
        assert rel_err(rs.linear_part, c["row_lin"]) <= tol, i
        pred = snx.predict(ds, x)
        if dtype == "f64":
            assert np.array_equal(pred, c["predict"]), i
        else:
            assert np.mean(pred != c["predict"]) <= 0.02, i
        seen += 1
    assert seen >= 5


def test_probs_sparse_and_torch_outputs():
    rng = np.random.default_rng(8)
    A = sp.random(500, 300, density=0.05, format="csr", random_state=8,
                  data_rvs=lambda k: rng.standard_normal(k))
    y = rng.integers(0, 20, 500)
    x = 0.3 * rng.standard_normal(19 * 300)
    D = A.toarray()
    ds = CsrDataset.from_scipy(A, y, 20)
    assert rel_err(snx.class_probabilities(ds, x), oracle.class_probs(D, y, 20, x)) <= 1e-10
    assert np.array_equal(snx.predict(ds, x), oracle.predict(D, y, 20, x))
    # device tensors in -> device tensors out
    xt = torch.from_numpy(x).cuda()
    assert isinstance(snx.predict(ds, xt), torch.Tensor)
    rs = snx.row_stats(ds, xt)
    assert isinstance(rs.max_part, torch.Tensor) and rs.max_part.shape == (500,)
