"""Inexact sub-sampled Newton-CG with Armijo line search (reference newton.py).

`minimize` is the generic loop and plugin seam (newton.py:60-112): any
objective_fn / oracle_factory pair works; vectors are kept on the device and
handed to foreign callables as numpy.  `newton_solve` (newton.py:115-140) is
the device-resident specialisation used for speed: x, g, p and the CG state
never leave HBM; the host only reads the scalars the reference branches on
(||g|| < eps, the Armijo test) and the trace values.

One deliberate fusion, output-identical to the reference: each line-search
trial F(x + a p) is a single pass that also counts correct predictions.  The
reference recomputes F at the accepted point (newton.py:98) -- that value is
bit-identical to the accepted trial (the trial point and the new iterate are
both formed by the same numpy-rounded x + a*p, snx_objective's `dir` path and
snx_axpy), so the trial's value and accuracy are reused instead of a third
full-data pass.
"""

import math
import os
import time
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import softmax
from .cg import CgConfig, cg_graph_for, cg_solve, report_from
from .device import AsyncRead, as_device, axpy, cuda_device, dot, download, vec_in, vec_out
from .errors import DataError, LineSearchError
from .linesearch import LineSearchConfig, line_search
from .sampling import SampleConfig, SubsampledOracle
from .trace import RunRecord, SolveTrace

VARIANT_FRACTIONS = {
    "full": (1.0, 1.0),
    "subsampled-100": (1.0, 0.05),
    "subsampled-20": (0.2, 0.05),
}


@dataclass(frozen=True)
class NewtonConfig:
    epsilon: float = 1e-8
    max_outer_iters: int = 100
    cg: CgConfig = field(default_factory=CgConfig)
    ls: LineSearchConfig = field(default_factory=LineSearchConfig)
    samples: SampleConfig = field(default_factory=SampleConfig)

    def __post_init__(self):
        if self.epsilon <= 0:
            raise DataError(f"epsilon must be > 0, got {self.epsilon}")


def make_variant(name, base=NewtonConfig()):
    """NewtonConfig with the named variant's sample fractions (newton.py:46-57)."""
    if name not in VARIANT_FRACTIONS:
        raise ValueError(
            f"unknown variant {name!r}; expected one of {sorted(VARIANT_FRACTIONS)}")
    f_g, f_h = VARIANT_FRACTIONS[name]
    return replace(base, samples=replace(base.samples, gradient_fraction=f_g,
                                         hessian_fraction=f_h))


def _host(v):
    return v.cpu().numpy()


def minimize(objective_fn, oracle_factory, x0, cfg, metrics=None, solver_name="newton"):
    """Generic inexact Newton-CG loop (newton.py:60-112).

    oracle_factory(k) -> object with .gradient(x) and .hessian_operator(x);
    objective_fn(x) -> full objective; metrics(x) -> (train_acc, test_acc).
    Callables flagged `_snx_device` receive device tensors, others numpy.
    """
    n0 = x0.numel() if isinstance(x0, torch.Tensor) else len(np.asarray(x0))
    x, as_t = vec_in(x0, n0, "initial point")
    x = x.clone()
    on_dev = lambda fn: getattr(fn, "_snx_device", False)  # noqa: E731
    f_dev = on_dev(objective_fn)

    def F(v):
        return float(objective_fn(v if f_dev else _host(v)))

    def M(v):
        if metrics is None:
            return math.nan, math.nan
        return metrics(v if on_dev(metrics) else _host(v))

    t0 = time.perf_counter()
    f_cur = F(x)
    tr, te = M(x)
    records = [RunRecord(solver_name, 0, 0.0, f_cur, tr, te, 0.0, 0)]
    reason = "max-iters"
    for k in range(cfg.max_outer_iters):
        oracle = oracle_factory(k)
        xin = x if on_dev(oracle) else _host(x)
        g, _ = vec_in(oracle.gradient(xin), n0, "gradient")
        if math.sqrt(float(dot(g, g))) < cfg.epsilon:
            reason = "gradient-converged"
            break
        report = cg_solve(oracle.hessian_operator(xin), g, cfg.cg)
        p = report.solution
        slope = float(dot(p, g))
        try:
            alpha, _ = line_search(lambda a: F(axpy(x, a, p)), f_cur, slope, cfg.ls)
        except LineSearchError:
            reason = "line-search-failure"
            break
        x = axpy(x, alpha, p)
        f_cur = F(x)
        tr, te = M(x)
        records.append(RunRecord(solver_name, k + 1, time.perf_counter() - t0, f_cur, tr, te,
                                 alpha, report.iterations))
    return SolveTrace(records, vec_out(x, as_t), reason)


class _Trial:
    """F(x + a p) and the correct count at that point, one fused device pass;
    the first trial (a = alpha0) may be pre-evaluated (speculative pipeline)."""

    def __init__(self, view, lam, x, p, first=None):
        self.view, self.lam, self.x, self.p = view, lam, x, p
        self.seen = {}
        if first is not None:
            self.seen[first[0]] = first[1:]

    def __call__(self, a):
        hit = self.seen.get(a)
        if hit is not None:
            return hit[0]
        out, corr = softmax.objective_parts(self.view, self.x, self.p, a, want_correct=True)
        loss, wsq = out.tolist()
        f = loss + 0.5 * self.lam * wsq
        self.seen[a] = (f, int(corr))
        return f


def newton_solve(prob, cfg, x0=None, test_set=None, solver_name="newton"):
    """Sub-sampled Newton-CG on a SoftmaxProblem, device resident (newton.py:115-140).

    x0 defaults to zeros.  Rows log the full objective, train accuracy and,
    with a test set, test accuracy.  x0 may be numpy (x_final is numpy) or a
    CUDA tensor (x_final stays on the device).

    Each outer iteration is enqueued as one pipeline read back with a single
    wait: gradient, ||g||^2, the Hessian sample and the captured CG solve, the
    slope p.g and the first Armijo trial at x + alpha0 p (with a full gradient
    sample the fused objective + gradient + accuracy pass, so an accepted alpha0
    already yields the next gradient -- bit-identical to recomputing it).  While
    the host waits for iteration k's scalars, iteration k + 1 is already enqueued
    speculatively from x + alpha0 p: the GPU never idles through the host's
    Armijo / bookkeeping step.  When the line search picks another step (or the
    loop stops) the speculative work is discarded; its sample draw (the
    SubsampledOracle of k + 1) is kept for the re-launch from x + alpha p, and
    speculation pauses after a backtracked iteration (backtracking tends to
    repeat) until alpha0 is accepted again -- so a backtracking phase does not
    queue a whole wasted iteration in front of every Armijo trial.
    SNX_SPECULATE=always|never overrides this (A/B runs).  The decisions and the
    trace are the reference's (newton.py:80-104).
    """
    ds = as_device(prob.dataset)
    if ds.n_rows == 0:
        raise DataError("cannot solve on an empty dataset")
    n, d = ds.n_rows, ds.dim
    if x0 is None:
        x0 = np.zeros(d)
    x, as_t = vec_in(x0, d, "initial point")
    x = x.clone()
    test = as_device(test_set) if test_set is not None else None
    dev_prob = softmax.SoftmaxProblem(ds, prob.lam)
    lam = prob.lam
    a0 = cfg.ls.alpha0
    T = cfg.cg.max_iters

    def test_acc(w):
        return (float(softmax.correct_count(test, w)) / test.n_rows) if test is not None \
            else math.nan

    def launch(k, oracle, x, g):
        """Enqueue iteration k at (x, g); nothing is read back yet."""
        if g is None:
            g = oracle.gradient_device(x)[0]
        gg = dot(g, g)
        hess = oracle.hessian_operator(x)
        cgws = cg_graph_for(hess, T, cfg.cg.theta).run(g)
        p = cgws.pb.clone()
        slope_t = dot(p, g)
        x_try = axpy(x, a0, p)
        fused = softmax.gradient_and_correct(ds, x_try, 1.0, lam) \
            if oracle.gradient_is_full else None
        if fused is not None:
            g_try, out_t, corr_t = fused
        else:
            g_try = None
            out_t, corr_t = softmax.objective_parts(ds, x_try, want_correct=True)
        reads = [gg, slope_t, out_t, corr_t, cgws.slot(T)]
        if test is not None:
            reads.append(softmax.correct_count(test, x_try))
        return {"p": p, "x_try": x_try, "g_try": g_try, "read": AsyncRead(*reads),
                "cgws": cgws, "oracle": oracle}

    policy = os.environ.get("SNX_SPECULATE", "adaptive")
    speculate = policy != "never"
    t0 = time.perf_counter()
    out, corr = softmax.objective_parts(ds, x, want_correct=True)
    loss, wsq = out.tolist()
    f_cur = loss + 0.5 * lam * wsq
    records = [RunRecord(solver_name, 0, 0.0, f_cur, int(corr) / n, test_acc(x), 0.0, 0)]
    reason = "max-iters"
    cur = launch(0, SubsampledOracle(dev_prob, cfg.samples, 0), x, None) \
        if cfg.max_outer_iters > 0 else None
    for k in range(cfg.max_outer_iters):
        # speculate: iteration k + 1 from x + alpha0 p, before reading iteration k
        nxt = None
        orc_next = SubsampledOracle(dev_prob, cfg.samples, k + 1) \
            if k + 1 < cfg.max_outer_iters else None
        if orc_next is not None and speculate:
            nxt = launch(k + 1, orc_next, cur["x_try"], cur["g_try"])
        h = cur["read"].wait()
        h_gg, h_slope, h_out, h_corr, h_slot = h[:5]
        if math.sqrt(float(h_gg)) < cfg.epsilon:
            reason = "gradient-converged"
            break
        report = report_from(cur["cgws"], T, True, slot_values=h_slot.tolist())
        p = cur["p"]
        if int(report.iterations) == 0 and report.converged:
            p.zero_()  # cg.py:61-62
        f_try = float(h_out[0]) + 0.5 * lam * float(h_out[1])
        trial = _Trial(ds, lam, x, p, first=(a0, f_try, int(h_corr[0])))
        try:
            alpha, _ = line_search(trial, f_cur, float(h_slope), cfg.ls)
        except LineSearchError:
            reason = "line-search-failure"
            break
        if alpha == a0:
            x = cur["x_try"]  # the same numpy-rounded x + a0 p (snx_axpy)
            te = float(h[5][0]) / test.n_rows if test is not None else math.nan
            g_next = cur["g_try"]
            cur = nxt  # the speculation holds (None when it was paused)
            if cur is None and orc_next is not None:
                cur = launch(k + 1, orc_next, x, g_next)
            speculate = policy != "never"
        else:
            x = axpy(x, alpha, p)
            te = test_acc(x)
            cur = launch(k + 1, orc_next, x, None) if orc_next is not None else None
            speculate = policy == "always"
        f_cur, ncorr = trial.seen[alpha]
        records.append(RunRecord(solver_name, k + 1, time.perf_counter() - t0, f_cur,
                                 ncorr / n, te, alpha, report.iterations))
    return SolveTrace(records, vec_out(x, as_t), reason)
