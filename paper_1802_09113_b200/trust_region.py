"""Sub-sampled trust-region Newton with Steihaug-CG (BASELINE config #4).

The reference has no trust-region solver (SPEC.md:409 lists it as a
non-goal), so this follows the CPU restatement in oracle/trust_region.py,
itself N&W Alg. 7.2 (Steihaug-CG) + Alg. 4.1 (radius update): PARITY
UNPINNED against the reference, pinned against the restatement by the GPU
tests.  Steihaug-CG is device resident (snx_tr_init / snx_tr_update: every
branch of Alg. 7.2 decided on the device from fixed-order reductions, the
whole solve captured as one CUDA graph); the host makes the outer radius /
acceptance decisions (Alg. 4.1) once per iteration.
"""

import gc
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, softmax
from .cg import _EAGER
from .device import (as_device, axpy, cuda_device, dot, download, ptr, stream_handle, vec_in,
                     vec_out)
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


class TrWorkspace:
    """Device buffers of one Steihaug-CG solve (d-vectors z, r, d, Hd, z_next,
    the CG-slot state and the radius as a device scalar)."""

    def __init__(self, d, T, device):
        f64 = dict(dtype=torch.float64, device=device)
        self.d, self.T = d, T
        self.vecs = torch.empty((5, d), **f64)
        self.z, self.r, self.dv, self.Hd, self.znew = self.vecs
        self.state = torch.zeros((T + 2) * _lib.CG_SLOT + 4 * _lib.DOT_BLOCKS, **f64)
        self.dots = torch.empty(2 * _lib.DOT_BLOCKS, **f64)
        self.radius = torch.zeros(1, **f64)
        self.g = torch.zeros(d, **f64)

    def slot(self, t):
        return self.state[t * _lib.CG_SLOT:(t + 1) * _lib.CG_SLOT]

    def done_ptr(self, t):
        return ptr(self.state) + (t * _lib.CG_SLOT + 1) * 8


def enqueue_steihaug(op, ws, theta):
    """snx_tr_init + T x (Hessian product of d, snx_tr_update): no host round trip."""
    _lib.call("snx_tr_init", ptr(ws.g), ws.d, float(theta), ws.T, ptr(ws.z), ptr(ws.r),
              ptr(ws.dv), ptr(ws.state), stream_handle())
    for t in range(ws.T):
        op.apply_into(ws.dv, ws.Hd, dots=ws.dots, skip=ws.done_ptr(t))
        _lib.call("snx_tr_update", t, ws.T, ws.d, ptr(ws.radius), ptr(ws.Hd), ptr(ws.dots),
                  ptr(ws.z), ptr(ws.r), ptr(ws.dv), ptr(ws.znew), ptr(ws.state), stream_handle())


class SteihaugGraph:
    """The whole Steihaug-CG solve captured once per operator buffers (like
    cg.CgGraph): inputs g and the radius are copied into the captured buffers."""

    def __init__(self, op, d, T, theta, device):
        self.op, self.theta = op, float(theta)
        self.ws = TrWorkspace(d, T, device)
        self.graph = None

    def run(self, g, radius):
        ws = self.ws
        ws.g.copy_(g)
        ws.radius.fill_(float(radius))
        if getattr(self.op, "_bufs", None) is None:  # foreign / sharded operator: eager
            enqueue_steihaug(self.op, ws, self.theta)
            return ws
        wsp = self.op.view.workspace(self.op.view.n_rows).data_ptr()
        if self.graph is not None and wsp != self._ws_ptr:
            self.graph = None
        if self.graph is None:
            self._ws_ptr = wsp
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                enqueue_steihaug(self.op, ws, self.theta)
            torch.cuda.current_stream().wait_stream(side)
            gc.collect()
            graph = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(graph, capture_error_mode="thread_local"):
                    enqueue_steihaug(self.op, ws, self.theta)
                self.graph = graph
            except RuntimeError:  # capture unsupported here: same kernels, eager launches
                torch.cuda.synchronize()
                self.graph = _EAGER
        if self.graph is _EAGER:
            enqueue_steihaug(self.op, ws, self.theta)
        else:
            self.graph.replay()
        return ws


def steihaug_graph_for(op, T, theta):
    hb = getattr(op, "_bufs", None)
    if hb is None:
        return SteihaugGraph(op, op.dim, T, theta, cuda_device())
    key = ("steihaug", T, float(theta), op.scale, op.lam, op.dim)
    g = hb.graphs.get(key)
    if g is None:
        g = hb.graphs[key] = SteihaugGraph(op, op.dim, T, theta, hb.h.device)
    g.op = op
    if hb.owner is not op:
        op._prepare()
    return g


def steihaug_cg(op, g, radius, theta, max_iters):
    """N&W Alg. 7.2 on the device; returns (p, m(p), iterations, on_boundary)."""
    ws = steihaug_graph_for(op, max_iters, theta).run(g, radius)
    st = ws.slot(max_iters).tolist()
    return ws.z.clone(), st[4], int(st[3]), st[2] != 0.0


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
    T = cfg.cg_max_iters
    g_next, oracle_next = None, None
    for k in range(cfg.max_outer_iters):
        # one host synchronisation per outer iteration: the gradient norm, the
        # Steihaug-CG result, F(x + p) (+ accuracy, + the gradient there when S_g
        # is the full set) and |p| are all enqueued before the host reads them
        oracle = oracle_next if oracle_next is not None else SubsampledOracle(dev_prob,
                                                                              cfg.samples, k)
        g = g_next if g_next is not None else oracle.gradient_device(x)[0]
        g_next = None
        gg = dot(g, g)
        op = oracle.hessian_operator(x)
        ws = steihaug_graph_for(op, T, cfg.theta).run(g, radius)
        step = ws.z.clone()
        x_try = axpy(x, 1.0, step)  # x + step
        fused = softmax.gradient_and_correct(ds, x_try, 1.0, prob.lam) \
            if oracle.gradient_is_full else None
        if fused is not None:
            g_try, out_t, corr_t = fused
        else:
            g_try = None
            out_t, corr_t = softmax.objective_parts(ds, x_try, want_correct=True)
        ss = dot(step, step)
        oracle_next = SubsampledOracle(dev_prob, cfg.samples, k + 1) \
            if k + 1 < cfg.max_outer_iters else None
        h_gg, h_out, h_corr, h_ss, h_slot = download(gg, out_t, corr_t, ss, ws.slot(T))
        if math.sqrt(float(h_gg)) < cfg.epsilon:
            reason = "gradient-converged"
            break
        m, iters, boundary = float(h_slot[4]), int(h_slot[3]), h_slot[2] != 0.0
        pred = -m
        f_trial = float(h_out[0]) + 0.5 * prob.lam * float(h_out[1])
        tr_trial = int(h_corr[0]) / n
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
            step_norm = math.sqrt(float(h_ss))
            x = x_try
            g_next = g_try
            f_cur, tr = f_trial, tr_trial
        records.append(RunRecord(solver_name, k + 1, time.perf_counter() - t0, f_cur, tr,
                                 test_acc(x), step_norm, iters))
        if radius < cfg.radius_min:
            reason = "radius-collapse"
            break
    return SolveTrace(records, vec_out(x, as_t), reason)
