"""Trust-region Newton with Steihaug-CG -- CPU restatement, TEST INFRASTRUCTURE.

PARITY UNPINNED: the reference has no trust-region solver (SPEC.md:409 lists
it as a non-goal).  The control flow follows the
literature the paper cites for Newton-CG ("nocedal2006numerical",
PAPER.md:216,728):

  * Steihaug-CG (Nocedal & Wright, Alg. 7.2) for  min g.p + 1/2 p.Hp, |p| <= Delta,
    stopping at |r| <= theta*|g| (the reference CG tolerance, cg.py:57-58),
  * radius update / acceptance of N&W Alg. 4.1 (rho < 1/4 shrinks by 1/4,
    rho > 3/4 on the boundary doubles up to Delta_max, accept iff rho > eta).

All arithmetic goes through the pinned pieces of ref_oracle (loss, grad,
hess_probs, hess_apply, draw_samples), so only this control flow is new.
The model decrease is tracked from CG scalars: m(z_{j+1}) = m(z_j) - a_j |r_j|^2
+ a_j^2 dHd_j / 2 (exact for CG iterates and for the boundary step, where
r_j.d_j = -|r_j|^2), so no extra Hessian product is spent on rho.
"""

import math
from dataclasses import dataclass

import numpy as np

from . import ref_oracle as ro


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


def _to_boundary(z, d, radius):
    """tau >= 0 with |z + tau d| = radius (positive root)."""
    dd = float(d @ d)
    zd = float(z @ d)
    zz = float(z @ z)
    disc = zd * zd + dd * (radius * radius - zz)
    return (-zd + math.sqrt(max(disc, 0.0))) / dd


def steihaug_cg(apply_H, g, radius, theta, max_iters):
    """N&W Alg. 7.2.  Returns (p, model_value m(p), iterations, hit_boundary)."""
    g = np.asarray(g, dtype=np.float64)
    gn = float(np.linalg.norm(g))
    z = np.zeros_like(g)
    if gn == 0.0:
        return z, 0.0, 0, False
    tol = theta * gn
    r = g.copy()
    d = -r
    rr = float(r @ r)
    m = 0.0
    for it in range(1, max_iters + 1):
        Hd = apply_H(d)
        dHd = float(d @ Hd)
        if dHd <= 0.0:
            tau = _to_boundary(z, d, radius)
            m += -tau * rr + 0.5 * tau * tau * dHd
            return z + tau * d, m, it, True
        a = rr / dHd
        z_next = z + a * d
        if float(np.linalg.norm(z_next)) >= radius:
            tau = _to_boundary(z, d, radius)
            m += -tau * rr + 0.5 * tau * tau * dHd
            return z + tau * d, m, it, True
        m += -a * rr + 0.5 * a * a * dHd
        z = z_next
        r = r + a * Hd
        rr_next = float(r @ r)
        if math.sqrt(rr_next) <= tol:
            return z, m, it, False
        d = -r + (rr_next / rr) * d
        rr = rr_next
    return z, m, max_iters, False


def trust_region_solve(A, y, C, lam, cfg=TrustRegionConfig(), gradient_fraction=1.0,
                       hessian_fraction=0.1, seed=0, x0=None, with_replacement=False):
    """Sub-sampled trust-region Newton (Hessian on S_H, n/|S_H| scale as sampling.py:82).

    Returns dict(records=[(k, f, train_acc, nan, step_norm, cg_iters, radius)], x, reason).
    """
    n, p = A.shape
    x = np.zeros((C - 1) * p) if x0 is None else np.array(x0, dtype=np.float64)
    f_cur = ro.loss(A, y, C, x, lam)
    radius = cfg.radius0
    records = [(0, f_cur, ro.accuracy(A, y, C, x), math.nan, 0.0, 0, radius)]
    reason = "max-iters"
    for k in range(cfg.max_outer_iters):
        s_g, s_h = ro.draw_samples(gradient_fraction, hessian_fraction, with_replacement,
                                   seed, n, k)
        full_g = len(s_g) == n and np.array_equal(s_g, np.arange(n))
        full_h = len(s_h) == n and np.array_equal(s_h, np.arange(n))
        Ag, yg = (A, y) if full_g else (A[s_g], y[s_g])
        Ah, yh = (A, y) if full_h else (A[s_h], y[s_h])
        g = ro.grad(Ag, yg, C, x, lam, scale=n / len(s_g))
        if np.linalg.norm(g) < cfg.epsilon:
            reason = "gradient-converged"
            break
        h = ro.hess_probs(Ah, yh, C, x)
        sh = n / len(s_h)
        step, m, iters, boundary = steihaug_cg(
            lambda v: ro.hess_apply(Ah, h, C, v, sh, lam), g, radius, cfg.theta,
            cfg.cg_max_iters)
        pred = -m
        f_trial = ro.loss(A, y, C, x + step, lam)
        rho = (f_cur - f_trial) / pred if pred > 0 else -math.inf
        if not np.isfinite(f_trial):
            rho = -math.inf
        if rho < 0.25:
            radius = 0.25 * radius
        elif rho > 0.75 and boundary:
            radius = min(2.0 * radius, cfg.radius_max)
        accepted = rho > cfg.eta
        if accepted:
            x = x + step
            f_cur = f_trial
        records.append((k + 1, f_cur, ro.accuracy(A, y, C, x), math.nan,
                        float(np.linalg.norm(step)) if accepted else 0.0, iters, radius))
        if radius < cfg.radius_min:
            reason = "radius-collapse"
            break
    return {"records": records, "x": x, "reason": reason}
