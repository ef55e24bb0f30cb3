"""CUDA path vs the reference (golden fixtures) and the CPU oracle.

Bars: fp64 path 1e-10 relative (north star), fp32 path 1e-4 relative
(declared separately), sample indices bit-exact, CG iteration counts and
Armijo step sizes exact, reruns bit-identical.
"""

import math

import numpy as np
import pytest
import torch

import oracle
import paper_1802_09113_b200 as snx
from conftest import rel_err, softmax_cases

pytestmark = pytest.mark.gpu

TOL64 = 1e-10
TOL32 = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _ds(A, y, C, dtype="f64"):
    return snx.DeviceDataset.from_numpy(A, y, C, dtype=dtype)


@pytest.mark.parametrize("dtype,tol", [("f64", TOL64), ("f32", TOL32)])
def test_softmax_golden(softmax_golden, dtype, tol):
    for i, c in softmax_cases(softmax_golden):
        n, p, C = (int(t) for t in c["shape"])
        if dtype == "f32" and i == 3:
            continue  # logits ~1e4: fp32 rounding of the logits alone exceeds 1e-4
        A, y, x, v, lam = c["A"], c["y"], c["x"], c["v"], float(c["lam"])
        ds = _ds(A, y, C, dtype)
        prob = snx.SoftmaxProblem(ds, lam)
        f = snx.objective(prob, x)
        ref = float(c["objective"])
        assert abs(f - ref) <= tol * max(1.0, abs(ref)), (i, f, ref)
        assert rel_err(snx.gradient(prob, x), c["gradient"]) <= tol, i
        op = snx.HessianOperator(ds, x, lam, scale=float(c["hess_scale"]))
        if n:
            assert rel_err(op._h.double().cpu().numpy(), c["hess_h"]) <= tol, i
        assert rel_err(op.apply(v), c["hess_apply"]) <= tol, i
        assert rel_err(op(v), c["hess_apply"]) <= tol, i
        assert rel_err(snx.hess_vec(prob, x, v), c["hess_vec"]) <= tol, i
        if n:
            acc = snx.accuracy(ds, x)
            if dtype == "f64":
                assert acc == float(c["accuracy"]), i
            else:
                assert abs(acc - float(c["accuracy"])) <= 2.0 / n
        else:
            with pytest.raises(snx.DataError):
                snx.accuracy(ds, x)


def test_dimension_errors(softmax_golden):
    c = dict(softmax_cases(softmax_golden))[0]
    ds = _ds(c["A"], c["y"], 4)
    prob = snx.SoftmaxProblem(ds, 0.0)
    with pytest.raises(snx.DimensionError):
        snx.objective(prob, np.zeros(5))
    with pytest.raises(snx.DimensionError):
        snx.HessianOperator(ds, c["x"], 0.0).apply(np.zeros(3))
    with pytest.raises(snx.DataError):
        snx.SoftmaxProblem(ds, -1.0)


def test_torch_in_torch_out(softmax_golden):
    c = dict(softmax_cases(softmax_golden))[6]
    ds = _ds(c["A"], c["y"], 10)
    prob = snx.SoftmaxProblem(ds, float(c["lam"]))
    xt = torch.from_numpy(c["x"]).cuda()
    g = snx.gradient(prob, xt)
    assert isinstance(g, torch.Tensor) and g.is_cuda
    assert rel_err(g.cpu().numpy(), c["gradient"]) <= TOL64


def test_reference_dataset_objects_accepted(softmax_golden):
    # duck-typed reference LabeledDataset (features.toarray(), labels, n_classes)
    c = dict(softmax_cases(softmax_golden))[1]

    class Feats:
        def __init__(self, A):
            self.A = A

        def toarray(self):
            return self.A

    class Labeled:
        def __init__(self, A, y, C):
            self.features, self.labels, self.n_classes = Feats(A), y, C

        @property
        def n_rows(self):
            return len(self.labels)

        @property
        def n_features(self):
            return self.features.A.shape[1]

    prob = snx.SoftmaxProblem(Labeled(c["A"], c["y"], 5), float(c["lam"]))
    assert abs(snx.objective(prob, c["x"]) - float(c["objective"])) <= TOL64 * abs(
        float(c["objective"]))


def test_sampled_oracle_indices_and_values(sampling_golden):
    n, p, C, lam = 50000, 32, 10, 1e-3
    A, y = oracle.synthetic_problem(n, p, C, seed=5)
    ds = _ds(A, y, C)
    prob = snx.SoftmaxProblem(ds, lam)
    cfg = snx.make_variant("subsampled-20").samples
    orc = snx.SubsampledOracle(prob, cfg, 0)
    ref_g, ref_h = oracle.draw_samples(0.2, 0.05, False, 0, n, 0)
    assert np.array_equal(orc.s_g, ref_g) and np.array_equal(orc.s_h, ref_h)
    assert np.array_equal(orc.s_h, sampling_golden["s0_s_h"])  # the reference's own draw
    x = 0.1 * np.random.default_rng(0).standard_normal((C - 1) * p)
    v = np.random.default_rng(1).standard_normal((C - 1) * p)
    g = orc.gradient(x)
    g_ref = oracle.grad(A[ref_g], y[ref_g], C, x, lam, scale=n / len(ref_g))
    assert rel_err(g, g_ref) <= TOL64
    h = oracle.hess_probs(A[ref_h], y[ref_h], C, x)
    hv_ref = oracle.hess_apply(A[ref_h], h, C, v, n / len(ref_h), lam)
    assert rel_err(orc.hess_vec(x, v), hv_ref) <= TOL64


def test_full_sample_is_unsampled_path():
    # f = 1 gives bit-identical results to the unsampled evaluation (test_sampling.py:73-86)
    n, p, C, lam = 300, 12, 5, 1e-3
    A, y = oracle.synthetic_problem(n, p, C, seed=9)
    ds = _ds(A, y, C)
    prob = snx.SoftmaxProblem(ds, lam)
    x = 0.2 * np.random.default_rng(4).standard_normal((C - 1) * p)
    v = np.random.default_rng(5).standard_normal((C - 1) * p)
    orc = snx.SubsampledOracle(prob, snx.SampleConfig(1.0, 1.0), 3)
    assert np.array_equal(orc.gradient(x), snx.gradient(prob, x))
    assert np.array_equal(orc.hess_vec(x, v),
                          snx.HessianOperator(ds, x, lam, scale=1.0).apply(v))


def test_cg_with_device_operator(solver_golden):
    g = solver_golden
    ds = _ds(g["cgh_A"], g["cgh_y"], 4)
    op = snx.HessianOperator(ds, g["cgh_x"], 1e-3, scale=2.0)
    rep = snx.cg_solve(op, g["cgh_g"], snx.CgConfig())
    assert rel_err(rep.solution, g["cgh_solution"]) <= 1e-9
    assert rep.iterations == int(g["cgh_stats"][1])
    assert rep.converged == bool(g["cgh_stats"][2])
    assert abs(rep.residual_norm - g["cgh_stats"][0]) <= 1e-8 * max(1.0, g["cgh_stats"][0])


def test_cg_with_foreign_operator(solver_golden):
    g = solver_golden
    for i in range(3):
        Q, rhs = g[f"cg{i}_Q"], g[f"cg{i}_g"]
        theta, iters = g[f"cg{i}_cfg"]
        calls = []

        def op(s, Q=Q):
            calls.append(1)
            return Q @ s

        rep = snx.cg_solve(op, rhs, snx.CgConfig(theta=float(theta), max_iters=int(iters)))
        ref = g[f"cg{i}_stats"]
        assert rel_err(rep.solution, g[f"cg{i}_solution"]) <= 1e-10
        assert rep.iterations == int(ref[1]) == len(calls)  # one application per iteration
        assert rep.converged == bool(ref[2])


def test_cg_zero_rhs_and_negative_curvature():
    rep = snx.cg_solve(lambda s: s, np.zeros(4), snx.CgConfig())
    assert rep.iterations == 0 and rep.converged and rep.residual_norm == 0.0
    assert np.array_equal(rep.solution, np.zeros(4))
    with pytest.raises(snx.CurvatureError):
        snx.cg_solve(lambda s: -s, np.ones(4), snx.CgConfig())


def test_newton_traces_match_reference(solver_golden):
    g = solver_golden
    for i in range(5):
        k = f"nt{i}_"
        n, p, C, seed, lam, iters, sseed = g[k + "params"]
        C, iters, sseed = int(C), int(iters), int(sseed)
        ds = _ds(g[k + "A"], g[k + "y"], C)
        test = _ds(g[k + "At"], g[k + "yt"], C) if k + "At" in g else None
        cfg = snx.make_variant(str(g[k + "variant"]), snx.NewtonConfig(
            max_outer_iters=iters, samples=snx.SampleConfig(seed=sseed)))
        tr = snx.newton_solve(snx.SoftmaxProblem(ds, float(lam)), cfg, test_set=test)
        ref = g[k + "records"]
        got = np.array([[r.iteration, r.objective, r.train_acc, r.test_acc, r.step_size,
                         r.cg_iters] for r in tr.records])
        assert got.shape == ref.shape, i
        assert np.array_equal(got[:, [0, 5]], ref[:, [0, 5]]), i  # iterations, CG iterations
        # Armijo step sizes are exact, except at the fp64 rounding floor: when the
        # reference backtracks below 1e-6 the sufficient-decrease margin
        # alpha*beta*|slope| is ~1e-13 |F|, i.e. ulp-level summation-order noise
        # decides; there only the objective (below) must agree.
        floor = (ref[:, 4] < 1e-6) & (ref[:, 0] > 0)
        assert np.array_equal(got[~floor, 4], ref[~floor, 4]), i
        assert np.array_equal(got[~floor, 2], ref[~floor, 2]), i
        assert np.allclose(got[:, 1], ref[:, 1], rtol=TOL64, atol=0), i
        assert np.array_equal(np.isnan(got[:, 3]), np.isnan(ref[:, 3]))
        fin = ~np.isnan(ref[:, 3])
        assert np.array_equal(got[fin, 3], ref[fin, 3])
        assert tr.reason == str(g[k + "reason"])
        assert rel_err(tr.x_final, g[k + "x_final"]) <= 1e-9, i


def test_newton_deterministic_reruns():
    A, y = oracle.synthetic_problem(3000, 40, 7, seed=11)
    ds = _ds(A, y, 7)
    prob = snx.SoftmaxProblem(ds, 1e-3)
    cfg = snx.make_variant("subsampled-20", snx.NewtonConfig(
        max_outer_iters=6, samples=snx.SampleConfig(seed=13)))
    a = snx.newton_solve(prob, cfg)
    b = snx.newton_solve(prob, cfg)
    assert np.array_equal(a.x_final, b.x_final)
    for ra, rb in zip(a.records, b.records):
        assert (ra.objective, ra.step_size, ra.cg_iters) == (rb.objective, rb.step_size,
                                                              rb.cg_iters)


def test_generic_minimize_with_foreign_oracle():
    # tests/test_newton.py:159-192: a plugin QuadraticOracle through minimize
    rng = np.random.default_rng(11)
    B = rng.standard_normal((6, 6))
    Q = B @ B.T + 6 * np.eye(6)
    b = rng.standard_normal(6)

    class QuadraticOracle:
        def gradient(self, x):
            return Q @ x + b

        def hessian_operator(self, x):
            return lambda v: Q @ v

    cfg = snx.NewtonConfig(epsilon=1e-10, max_outer_iters=10,
                           cg=snx.CgConfig(theta=1e-14, max_iters=50))
    tr = snx.minimize(lambda x: 0.5 * x @ (Q @ x) + b @ x, lambda k: QuadraticOracle(),
                      np.zeros(6), cfg)
    assert tr.reason == "gradient-converged" and tr.iterations == 1
    assert tr.records[1].step_size == 1.0
    assert np.allclose(tr.x_final, -np.linalg.solve(Q, b), rtol=1e-10)


@pytest.mark.parametrize("shape", [("mnist", 60000, 784, 10), ("cifar", 50000, 3072, 10),
                                   ("covertype", 581012, 54, 7)])
def test_benchmark_shapes_vs_oracle(shape):
    name, n, p, C = shape
    A, y = oracle.synthetic_problem(n, p, C, seed=0)
    lam = 1e-3
    for dtype, tol in (("f64", TOL64), ("f32", TOL32)):
        ds = _ds(A, y, C, dtype)
        prob = snx.SoftmaxProblem(ds, lam)
        x = 0.05 * np.random.default_rng(1).standard_normal((C - 1) * p)
        v = np.random.default_rng(2).standard_normal((C - 1) * p)
        orc = snx.SubsampledOracle(prob, snx.make_variant("subsampled-100").samples, 0)
        s_h = orc.s_h
        f = snx.objective(prob, x)
        f_ref = oracle.loss(A, y, C, x, lam)
        assert abs(f - f_ref) <= tol * abs(f_ref), (name, dtype)
        assert rel_err(orc.gradient(x), oracle.grad(A, y, C, x, lam)) <= tol, (name, dtype)
        h = oracle.hess_probs(A[s_h], y[s_h], C, x)
        hv_ref = oracle.hess_apply(A[s_h], h, C, v, n / len(s_h), lam)
        op = orc.hessian_operator(x)
        hv = op.apply(v)
        assert rel_err(hv, hv_ref) <= tol, (name, dtype, rel_err(hv, hv_ref))
        # size-independent properties: symmetry and linearity of the operator
        u = np.random.default_rng(3).standard_normal((C - 1) * p)
        hu = op.apply(u)
        assert abs(u @ hv - v @ hu) <= 10 * tol * abs(u @ hv)
        assert rel_err(op.apply(2.0 * v + u), 2.0 * hv + hu) <= 10 * tol
        acc = snx.accuracy(ds, x)
        acc_ref = oracle.accuracy(A, y, C, x)
        assert abs(acc - acc_ref) <= (0 if dtype == "f64" else 1e-4), (name, dtype)
        del ds
        torch.cuda.empty_cache()


def test_trust_region_matches_restatement():
    A, y = oracle.synthetic_problem(400, 12, 4, seed=3)
    cfg = oracle.TrustRegionConfig(max_outer_iters=12)
    ref = oracle.trust_region_solve(A, y, 4, 1e-3, cfg, hessian_fraction=0.1)
    ds = _ds(A, y, 4)
    tr = snx.trust_region_solve(snx.SoftmaxProblem(ds, 1e-3), snx.TrustRegionConfig(
        max_outer_iters=12, samples=snx.SampleConfig(1.0, 0.1)))
    assert len(tr.records) == len(ref["records"])
    for r, (k, f, acc, _, step, it, rad) in zip(tr.records, ref["records"]):
        assert r.iteration == k and r.cg_iters == it
        assert abs(r.objective - f) <= 1e-10 * abs(f)
        assert abs(r.step_size - step) <= 1e-8 * max(1.0, step)
    assert tr.reason == ref["reason"]
    assert rel_err(tr.x_final, ref["x"]) <= 1e-9
