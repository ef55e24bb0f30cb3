"""Pin the CPU oracle to the reference's own outputs (tests/golden/*.npz).

The fixtures were produced by tests/golden/make_golden.py running the
unmodified reference; the oracle must reproduce them before it may vouch
for the CUDA path.  fp64 parity bar: 1e-12 relative (same BLAS stack);
sample indices bit-exact.
"""

import math

import numpy as np
import pytest

import oracle
from conftest import rel_err, softmax_cases


def test_numpy_version_matches_fixture(sampling_golden):
    # Generator streams are only guaranteed within a numpy version.
    assert str(sampling_golden["meta_numpy"]) == np.__version__


def test_softmax_pieces(softmax_golden):
    seen = 0
    for i, c in softmax_cases(softmax_golden):
        n, p, C = (int(t) for t in c["shape"])
        A, y, x, v, lam = c["A"], c["y"], c["x"], c["v"], float(c["lam"])
        f = oracle.loss(A, y, C, x, lam)
        assert abs(f - float(c["objective"])) <= 1e-12 * max(1.0, abs(f)), i
        f0 = oracle.loss(A, y, C, np.zeros_like(x), lam)
        assert abs(f0 - n * math.log(C)) <= 1e-9 * max(1.0, f0)
        assert abs(f0 - float(c["objective0"])) <= 1e-12 * max(1.0, f0)
        assert rel_err(oracle.grad(A, y, C, x, lam), c["gradient"]) <= 1e-12, i
        h = oracle.hess_probs(A, y, C, x)
        assert rel_err(h, c["hess_h"]) <= 1e-13, i
        hv = oracle.hess_apply(A, h, C, v, float(c["hess_scale"]), lam)
        assert rel_err(hv, c["hess_apply"]) <= 1e-12, i
        hv1 = oracle.hess_apply(A, h, C, v, 1.0, lam)
        assert rel_err(hv1, c["hess_vec"]) <= 1e-12, i
        if n:
            assert rel_err(oracle.class_probs(A, y, C, x), c["probs"]) <= 1e-13
            assert np.array_equal(oracle.predict(A, y, C, x), c["predict"])
            assert oracle.accuracy(A, y, C, x) == float(c["accuracy"])
        seen += 1
    assert seen == 10


def test_sampling_bit_exact(sampling_golden):
    g = sampling_golden
    i = 0
    while f"s{i}_params" in g:
        fg, fh, rep, seed, n, it = g[f"s{i}_params"]
        n, it, seed = int(n), int(it), int(seed)
        s_g, s_h = oracle.draw_samples(fg, fh, bool(rep), seed, n, it)
        assert len(s_g) == int(g[f"s{i}_size_g"]) and len(s_h) == int(g[f"s{i}_size_h"])
        if bool(g[f"s{i}_s_g_full"]):
            assert np.array_equal(s_g, np.arange(n))
        else:
            assert np.array_equal(s_g, g[f"s{i}_s_g"])
        assert np.array_equal(s_h, g[f"s{i}_s_h"])
        i += 1
    assert i == 11


def test_survey_spot_values(sampling_golden):
    # first 8 / last 4 / sum of the CIFAR-shape S_H at k=0.
    s_h = oracle.draw_samples(1.0, 0.05, False, 0, 50000, 0)[1]
    assert list(s_h[:8]) == [5, 7, 8, 19, 72, 104, 110, 152]
    assert list(s_h[-4:]) == [49935, 49945, 49956, 49994]
    assert int(s_h.sum()) == 62171654
    # sample_size uses Python round (half to even): 0.05 * 581012 = 29050.6
    assert oracle.sample_size(0.05, 581012) == 29051


def test_cg(solver_golden):
    g = solver_golden
    for i in range(3):
        Q, rhs = g[f"cg{i}_Q"], g[f"cg{i}_g"]
        theta, iters = g[f"cg{i}_cfg"]
        sol, rn, it, conv = oracle.cg(lambda s: Q @ s, rhs, theta, int(iters))
        assert rel_err(sol, g[f"cg{i}_solution"]) <= 1e-12
        ref = g[f"cg{i}_stats"]
        assert it == int(ref[1]) and conv == bool(ref[2])
        assert abs(rn - ref[0]) <= 1e-12 * max(1.0, ref[0])
    A, y, x, rhs = g["cgh_A"], g["cgh_y"], g["cgh_x"], g["cgh_g"]
    h = oracle.hess_probs(A, y, 4, x)
    sol, rn, it, conv = oracle.cg(lambda s: oracle.hess_apply(A, h, 4, s, 2.0, 1e-3), rhs)
    assert rel_err(sol, g["cgh_solution"]) <= 1e-12
    assert it == int(g["cgh_stats"][1]) and conv == bool(g["cgh_stats"][2])


def test_line_search(solver_golden):
    g = solver_golden
    for i in range(3):
        vals = list(g[f"ls{i}_vals"])
        f0, slope, alpha, evals = g[f"ls{i}_result"]
        seq = iter(vals)
        a, e = oracle.armijo(lambda _a: next(seq), f0, slope)
        assert a == alpha and e == int(evals)
    with pytest.raises(oracle.ArmijoFailure):
        oracle.armijo(lambda a: 1.0, 1.0, 0.0)
    with pytest.raises(oracle.ArmijoFailure):
        oracle.armijo(lambda a: 2.0, 1.0, -1.0, max_iters=3)


def test_newton_traces(solver_golden):
    g = solver_golden
    for i in range(5):
        k = f"nt{i}_"
        variant = str(g[k + "variant"])
        n, p, C, seed, lam, iters, sseed = g[k + "params"]
        test = (g[k + "At"], g[k + "yt"]) if k + "At" in g else None
        out = oracle.newton_solve(g[k + "A"], g[k + "y"], int(C), float(lam), variant=variant,
                                  seed=int(sseed), max_outer_iters=int(iters), test=test)
        ref = g[k + "records"]
        got = np.array(out["records"], dtype=np.float64)
        assert got.shape == ref.shape
        assert np.array_equal(got[:, [0, 5]], ref[:, [0, 5]])          # iteration, cg_iters
        assert np.array_equal(got[:, 4], ref[:, 4])                    # step sizes (ladder)
        assert np.allclose(got[:, 1], ref[:, 1], rtol=1e-12, atol=0)   # objective
        assert np.array_equal(np.isnan(got[:, 3]), np.isnan(ref[:, 3]))
        assert out["reason"] == str(g[k + "reason"])
        assert rel_err(out["x"], g[k + "x_final"]) <= 1e-10


def test_lipschitz(solver_golden):
    g = solver_golden
    L = oracle.estimate_lipschitz(g["lip_A"], g["lip_y"], 3, iters=50)
    assert abs(L - float(g["lip_L"])) <= 1e-12 * abs(L)


def test_trust_region_oracle_descends():
    # parity unpinned (no reference TR); check its own invariants instead.
    A, y = oracle.synthetic_problem(400, 12, 4, seed=3, normalize=True)
    out = oracle.trust_region_solve(A, y, 4, 1e-3,
                                    oracle.TrustRegionConfig(max_outer_iters=15),
                                    hessian_fraction=0.1)
    f = np.array([r[1] for r in out["records"]])
    assert np.all(np.diff(f) <= 1e-12)
    assert f[-1] < f[0]
    g = oracle.grad(A, y, 4, out["x"], 1e-3)
    assert np.linalg.norm(g) < np.linalg.norm(oracle.grad(A, y, 4, np.zeros(36), 1e-3))
