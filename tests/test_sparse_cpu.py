"""The dense oracle restatement reproduces the reference's CSR-storage results
(the reference's own claim: dense and sparse products agree to <= 1e-12,
dataset.py:24-26), so one oracle pins both storages."""

import numpy as np

import oracle
from conftest import rel_err, sparse_cases


def test_oracle_matches_reference_sparse(sparse_golden):
    n_cases = 0
    for i, A, C, c in sparse_cases(sparse_golden):
        D = A.toarray()
        y, x, v = c["y"], c["x"], c["v"]
        assert abs(oracle.loss(D, y, C, x, 1e-3) - float(c["objective"])) <= 1e-12 * abs(
            float(c["objective"]))
        assert rel_err(oracle.grad(D, y, C, x, 1e-3), c["gradient"]) <= 1e-12
        h = oracle.hess_probs(D, y, C, x)
        assert rel_err(oracle.hess_apply(D, h, C, v, 3.0, 1e-3), c["hess_apply"]) <= 1e-12
        assert oracle.accuracy(D, y, C, x) == float(c["accuracy"])
        n_cases += 1
    assert n_cases == 4
