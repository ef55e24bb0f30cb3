"""Conjugate gradient for H p = -g with best-iterate tracking (reference cg.py).

The CG state (r, s, p, p_best and the scalars rs, ||r_best||, threshold,
iteration count, flags) lives on the device.  One iteration is

    snx_hess_apply(s -> Hs, + s.Hs / s.s partials)   [skipped once done]
    snx_cg_update(t)  = curvature test, alpha, p/r update, best copy, stop
                        test and new direction (cg.py:77-96)

so the whole solve is enqueued without a host round trip; the host reads the
final slot once.  Every decision (curvature <= 1e-32 s.s, r_norm <= best,
r_norm <= theta ||g||) is the reference's, taken on device in fp64.

Foreign operators (any callable v -> H v, e.g. the reference's own
HessianOperator or a test's CountingOperator, tests/test_cg.py:10-20) are
supported through the same device state: s is handed to the callable as
numpy and H s uploaded back.
"""

import gc
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import cuda_device, download, ptr, stream_handle, vec_in, vec_out
from .errors import CurvatureError, DataError

CURVATURE_EPS = 1e-32  # cg.py:16


@dataclass(frozen=True)
class CgConfig:
    """theta: relative residual tolerance; max_iters: operator applications."""

    theta: float = 1e-4
    max_iters: int = 10

    def __post_init__(self):
        if not 0.0 < self.theta < 1.0:
            raise DataError(f"theta must be in (0, 1), got {self.theta}")
        if self.max_iters < 1:
            raise DataError(f"max_iters must be >= 1, got {self.max_iters}")


@dataclass
class CgReport:
    """solution = best iterate by residual norm (or -g when nothing improved)."""

    solution: object
    residual_norm: float
    iterations: int
    converged: bool


class CgWorkspace:
    """Device buffers of one CG solve of dimension d with at most T iterations."""

    def __init__(self, d, T, device):
        f64 = dict(dtype=torch.float64, device=device)
        self.d, self.T = d, T
        self.vecs = torch.empty((5, d), **f64)
        self.r, self.s, self.p, self.pb, self.Hs = self.vecs
        # slots + two scratch rows of block partials (r.r, and s.s for the fused update)
        self.state = torch.zeros((T + 2) * _lib.CG_SLOT + 2 * _lib.DOT_BLOCKS, **f64)
        self.dots = torch.empty(2 * _lib.DOT_BLOCKS, **f64)

    def slot(self, t):
        return self.state[t * _lib.CG_SLOT:(t + 1) * _lib.CG_SLOT]

    def done_ptr(self, t):
        return _lib.done_flag(ptr(self.state), t)


def enqueue_cg(op, g, theta, T, ws):
    """Enqueue init + T iterations with a device operator (op.apply_into)."""
    d = ws.d
    _lib.call("snx_cg_init", ptr(g), d, float(theta), T, ptr(ws.r), ptr(ws.s), ptr(ws.p),
              ptr(ws.pb), ptr(ws.state), stream_handle())
    fused = getattr(op, "apply_cg_into", None)
    for t in range(T):
        if fused is not None and fused(t, T, ws):  # product + CG update, finalize fused
            continue
        op.apply_into(ws.s, ws.Hs, dots=ws.dots, skip=ws.done_ptr(t))
        _lib.call("snx_cg_update", t, T, d, ptr(ws.Hs), ptr(ws.dots), ptr(ws.r), ptr(ws.s),
                  ptr(ws.p), ptr(ws.pb), ptr(ws.state), stream_handle())


_EAGER = object()  # marker: graph capture failed, launch eagerly


class CgGraph:
    """The whole device CG solve (init + T iterations, ~6T kernels) captured
    once as a CUDA graph for an operator's shared sample buffers; replayed
    every outer iteration (launch overhead ~1 us per node instead of ~4 us per
    stream launch).  Inputs: `g` (copied into self.g); outputs: ws."""

    def __init__(self, op, d, T, theta, device):
        self.op, self.T, self.theta = op, T, float(theta)
        self.g = torch.zeros(d, dtype=torch.float64, device=device)
        self.ws = CgWorkspace(d, T, device)
        self.graph = None

    def _enqueue(self):
        enqueue_cg(self.op, self.g, self.theta, self.T, self.ws)

    def run(self, g):
        """g: the right-hand side (device tensor), or None when self.g already
        holds it."""
        if g is not None:
            self.g.copy_(g)
        ws_now = self.op.view.workspace(self.op.view.n_rows).data_ptr()
        if self.graph is not None and ws_now != self._ws_ptr:
            self.graph = None  # the dataset workspace moved: recapture
        if self.graph is None:
            self._ws_ptr = ws_now
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):  # warm-up: kernel attributes, workspace
                self._enqueue()
            torch.cuda.current_stream().wait_stream(side)
            # collect garbage first: a CUDA graph freed by the GC in the middle of
            # this capture would invalidate it
            gc.collect()
            graph = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(graph, capture_error_mode="thread_local"):
                    self._enqueue()
                self.graph = graph
            except RuntimeError:  # capture unsupported here: same kernels, eager launches
                torch.cuda.synchronize()
                self.graph = _EAGER
        if self.graph is _EAGER:
            self._enqueue()
        else:
            self.graph.replay()
        return self.ws


def cg_graph_for(op, T, theta):
    """The CgGraph of op's shared buffers for (T, theta, scale, lam)."""
    hb = op._bufs
    key = (T, float(theta), op.scale, op.lam, op.dim)
    cg = hb.graphs.get(key)
    if cg is None:
        cg = hb.graphs[key] = CgGraph(op, op.dim, T, theta, hb.h.device)
    cg.op = op
    if hb.owner is not op:
        op._prepare()
    return cg


def _foreign_loop(apply_H, T, ws):
    d = ws.d
    last = 0
    for t in range(T):
        if float(ws.slot(t)[2]) != 0.0:  # done: the operator is host code anyway
            return t
        hs = apply_H(ws.s.cpu().numpy())
        hs = np.asarray(hs, dtype=np.float64)
        ws.Hs.copy_(torch.from_numpy(np.ascontiguousarray(hs)))
        _lib.call("snx_dot_partials", ptr(ws.s), ptr(ws.Hs), d, ptr(ws.dots), stream_handle())
        _lib.call("snx_dot_partials", ptr(ws.s), ptr(ws.s), d,
                  ptr(ws.dots) + 8 * _lib.DOT_BLOCKS, stream_handle())
        _lib.call("snx_cg_update", t, T, d, ptr(ws.Hs), ptr(ws.dots), ptr(ws.r), ptr(ws.s),
                  ptr(ws.p), ptr(ws.pb), ptr(ws.state), stream_handle())
        last = t + 1
    return last


def report_from(ws, t_final, as_torch, slot_values=None):
    """CgReport of a finished device solve; slot_values: the final slot already
    read by the caller (no extra synchronisation; the solution is ws.pb)."""
    if slot_values is not None:
        st = list(slot_values)
        sol = ws.pb
    elif as_torch:
        st = ws.slot(t_final).tolist()
        sol = ws.pb.clone()
    else:  # one synchronisation for the scalars and the solution
        st, sol = download(ws.slot(t_final), ws.pb)
        st = st.tolist()
    rs, best, done, iters, conv, thr, err, curv = st
    if err != 0.0:
        raise CurvatureError(
            f"non-positive curvature s^T H s = {curv:.3e} at CG iteration {int(iters)}; "
            "operator is not positive definite")
    if int(iters) == 0 and conv != 0.0:
        sol = torch.zeros_like(sol) if as_torch else np.zeros_like(sol)  # cg.py:61-62: zeros for g == 0
    return CgReport(sol, best, int(iters), bool(conv))


def cg_solve(apply_H, g, cfg):
    """Approximately solve H p = -g to ||H p + g|| <= theta ||g|| (cg.py:51-98)."""
    if getattr(apply_H, "_bufs", None) is not None and not isinstance(g, torch.Tensor):
        a = np.ascontiguousarray(g, dtype=np.float64)
        cg = cg_graph_for(apply_H, cfg.max_iters, cfg.theta)
        if a.ndim == 1 and a.shape[0] == cg.g.numel():
            # numpy g straight into the captured graph's input (one async copy)
            cg.g.copy_(torch.from_numpy(a), non_blocking=True)
            return report_from(cg.run(None), cfg.max_iters, False)
    gd, as_t = vec_in(g, np.asarray(g).shape[0] if not isinstance(g, torch.Tensor)
                      else g.numel(), "gradient")
    if getattr(apply_H, "_bufs", None) is not None:  # our operator: graph-captured solve
        ws = cg_graph_for(apply_H, cfg.max_iters, cfg.theta).run(gd)
        return report_from(ws, cfg.max_iters, as_t)
    ws = CgWorkspace(gd.numel(), cfg.max_iters, cuda_device())
    if getattr(apply_H, "_snx_device", False):
        enqueue_cg(apply_H, gd, cfg.theta, cfg.max_iters, ws)
        t_final = cfg.max_iters
    else:
        _lib.call("snx_cg_init", ptr(gd), ws.d, float(cfg.theta), cfg.max_iters, ptr(ws.r),
                  ptr(ws.s), ptr(ws.p), ptr(ws.pb), ptr(ws.state), stream_handle())
        t_final = _foreign_loop(apply_H, cfg.max_iters, ws)
    return report_from(ws, t_final, as_t)
