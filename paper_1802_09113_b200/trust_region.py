"""Sub-sampled trust-region Newton with Steihaug-CG (BASELINE config #4).

The reference has no trust-region solver (SPEC.md:409 lists it as a
non-goal), so this follows the CPU restatement in oracle/trust_region.py,
itself N&W Alg. 7.2 (Steihaug-CG) + Alg. 4.1 (radius update): PARITY
UNPINNED against the reference, pinned against the restatement by the GPU
tests.  All vector work is device-resident (Hessian products through
snx_hess_apply, updates through snx_axpy/snx_axpby, norms through the
fixed-order snx_dot); the host makes the scalar decisions.
"""

import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import softmax
from .device import as_device, axpby, axpy, dot, vec_in, vec_out
from .errors import DataError
from .sampling import SampleConfig, SubsampledOracle
from .trace import RunRecord, SolveTrace


@dataclass(frozen=True)
class TrustRegionConfig:
    radius0: float = 1.0
    radius_max: float = 1e3
    eta: float = 0.1
    theta: float = 1e-4
    cg_max_iters: int = 10
    epsilon: float = 1e-8
    max_outer_iters: int = 100
    radius_min: float = 1e-12
    samples: SampleConfig = field(
        default_factory=lambda: SampleConfig(gradient_fraction=1.0, hessian_fraction=0.1))

    def __post_init__(self):
        if not 0.0 < self.radius0 <= self.radius_max:
            raise DataError("need 0 < radius0 <= radius_max")
        if not 0.0 <= self.eta < 0.25:
            raise DataError(f"eta must be in [0, 1/4), got {self.eta}")
        if not 0.0 < self.theta < 1.0 or self.cg_max_iters < 1:
            raise DataError("theta must be in (0, 1) and cg_max_iters >= 1")


def _scalars(*pairs):
    """Several fixed-order device dots, one host synchronisation."""
    return torch.stack([dot(a, b) for a, b in pairs]).tolist()


def _to_boundary(z, d, radius):
    dd, zd, zz = _scalars((d, d), (z, d), (z, z))
    disc = zd * zd + dd * (radius * radius - zz)
    return (-zd + math.sqrt(max(disc, 0.0))) / dd


def steihaug_cg(op, g, radius, theta, max_iters):
    """N&W Alg. 7.2 on device vectors; returns (p, m(p), iterations, on_boundary)."""
    gn = math.sqrt(float(dot(g, g)))
    z = torch.zeros_like(g)
    if gn == 0.0:
        return z, 0.0, 0, False
    tol = theta * gn
    r = g.clone()
    dvec = axpby(-1.0, g, 0.0, g)  # d0 = -r0 = -g
    Hd = torch.empty_like(g)
    rr = gn * gn
    m = 0.0
    for it in range(1, max_iters + 1):
        op.apply_into(dvec, Hd)
        dHd = float(dot(dvec, Hd))
        if dHd <= 0.0:
            tau = _to_boundary(z, dvec, radius)
            m += -tau * rr + 0.5 * tau * tau * dHd
            return axpy(z, tau, dvec), m, it, True
        a = rr / dHd
        z_next = axpy(z, a, dvec)
        if math.sqrt(float(dot(z_next, z_next))) >= radius:
            tau = _to_boundary(z, dvec, radius)
            m += -tau * rr + 0.5 * tau * tau * dHd
            return axpy(z, tau, dvec), m, it, True
        m += -a * rr + 0.5 * a * a * dHd
        z = z_next
        r = axpy(r, a, Hd)
        rr_next = float(dot(r, r))
        if math.sqrt(rr_next) <= tol:
            return z, m, it, False
        dvec = axpby(-1.0, r, rr_next / rr, dvec)
        rr = rr_next
    return z, m, max_iters, False


def trust_region_solve(prob, cfg=TrustRegionConfig(), x0=None, test_set=None,
                       solver_name="trust-region"):
    """Trace rows: step_size = ||p|| of an accepted step (0 when rejected)."""
    ds = as_device(prob.dataset)
    if ds.n_rows == 0:
        raise DataError("cannot solve on an empty dataset")
    n, d = ds.n_rows, ds.dim
    x, as_t = vec_in(np.zeros(d) if x0 is None else x0, d, "initial point")
    x = x.clone()
    test = as_device(test_set) if test_set is not None else None
    dev_prob = softmax.SoftmaxProblem(ds, prob.lam)

    def f_and_acc(w, direction=None, alpha=0.0):
        out, corr = softmax.objective_parts(ds, w, direction, alpha, want_correct=True)
        loss, wsq = out.tolist()
        return loss + 0.5 * prob.lam * wsq, int(corr) / n

    def test_acc(w):
        return float(softmax.correct_count(test, w)) / test.n_rows if test else math.nan

    t0 = time.perf_counter()
    f_cur, tr = f_and_acc(x)
    radius = cfg.radius0
    records = [RunRecord(solver_name, 0, 0.0, f_cur, tr, test_acc(x), 0.0, 0)]
    reason = "max-iters"
    for k in range(cfg.max_outer_iters):
        oracle = SubsampledOracle(dev_prob, cfg.samples, k)
        g, _ = oracle.gradient_device(x)
        if math.sqrt(float(dot(g, g))) < cfg.epsilon:
            reason = "gradient-converged"
            break
        op = oracle.hessian_operator(x)
        step, m, iters, boundary = steihaug_cg(op, g, radius, cfg.theta, cfg.cg_max_iters)
        pred = -m
        f_trial, tr_trial = f_and_acc(x, step, 1.0)
        rho = (f_cur - f_trial) / pred if pred > 0 else -math.inf
        if not np.isfinite(f_trial):
            rho = -math.inf
        if rho < 0.25:
            radius = 0.25 * radius
        elif rho > 0.75 and boundary:
            radius = min(2.0 * radius, cfg.radius_max)
        accepted = rho > cfg.eta
        step_norm = 0.0
        if accepted:
            step_norm = math.sqrt(float(dot(step, step)))
            x = axpy(x, 1.0, step)
            f_cur, tr = f_trial, tr_trial
        records.append(RunRecord(solver_name, k + 1, time.perf_counter() - t0, f_cur, tr,
                                 test_acc(x), step_norm, iters))
        if radius < cfg.radius_min:
            reason = "radius-collapse"
            break
    return SolveTrace(records, vec_out(x, as_t), reason)
