"""Row-sharded multi-GPU sub-sampled Newton-CG.

The reference is single-process (SPEC.md:409 lists distribution as a
non-goal).  Every data term of the method is a sum over rows
(softmax.py:130-134, 154-162, 203-209), so rows shard naturally:

  * rank r of W holds the contiguous rows [n*r/W, n*(r+1)/W) in HBM;
  * the sample sets S_g, S_H are drawn GLOBALLY on every rank with the
    reference's numpy streams (bit-identical on all ranks) and each rank
    keeps the indices inside its shard (searchsorted on the sorted set);
  * gradient and Hessian products are computed per shard with lam = 0, summed
    over ranks with ONE NCCL all-reduce of the d-vector, and finished with
    lam * x (snx_finish_hv also emits the CG dot partials of the summed
    vector); objective / accuracy all-reduce two scalars;
  * the CG state (d-vectors) is replicated: every rank sees the same summed
    H s, so the CG scalars need no extra collective.

torch.distributed owns the process group (one process per GPU, NCCL over
NVLink); the arithmetic is libsnx's.
"""

import math
import time

import numpy as np
import torch
import torch.distributed as dist

from . import _lib, softmax
from .cg import CgWorkspace, enqueue_cg, report_from
from .device import (DeviceDataset, as_device, axpy, dot, download, ptr, stream_handle, vec_in,
                     vec_out)
from .errors import DataError, LineSearchError
from .linesearch import line_search
from .sampling import draw_samples, sample_size
from .trace import RunRecord, SolveTrace


def shard_bounds(n, world, rank):
    """Contiguous row range [lo, hi) of `rank` (balanced to within one row)."""
    return n * rank // world, n * (rank + 1) // world


def local_indices(sample, lo, hi):
    """The part of a sorted global sample inside [lo, hi), as shard-local indices."""
    s = np.asarray(sample, dtype=np.int64)
    a, b = np.searchsorted(s, [lo, hi], side="left")
    return s[a:b] - lo


def world_info(group=None):
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def all_reduce_(t, group=None):
    """In-place sum over ranks (identity when not distributed)."""
    if world_info(group)[0] > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


class ShardedProblem:
    """This rank's shard of a global L2-regularised softmax problem."""

    def __init__(self, local, n_global, row0, lam, group=None):
        if lam < 0:
            raise DataError(f"regularization coefficient must be >= 0, got {lam}")
        self.local = as_device(local)
        self.n_global = int(n_global)
        self.row0 = int(row0)
        self.lam = float(lam)
        self.group = group

    @classmethod
    def from_global(cls, features, labels, n_classes, lam, dtype="f64", group=None):
        """Upload only this rank's rows of a host dataset."""
        world, rank = world_info(group)
        n = len(labels)
        lo, hi = shard_bounds(n, world, rank)
        local = DeviceDataset.from_numpy(features[lo:hi], labels[lo:hi], n_classes, dtype=dtype)
        return cls(local, n, lo, lam, group)

    @property
    def dim(self):
        return self.local.dim

    @property
    def row1(self):
        return self.row0 + self.local.n_rows

    def objective_parts_device(self, w, direction=None, alpha=0.0):
        """Device [global data loss, global #correct] (one all-reduce of two
        scalars) and the local [loss, ||w_eff||^2] (the norm is replicated)."""
        out, corr = softmax.objective_parts(self.local, w, direction, alpha, want_correct=True)
        buf = torch.stack([out[0], corr[0].to(torch.float64)])
        all_reduce_(buf, self.group)
        return buf, out

    def objective_and_correct(self, w, direction=None, alpha=0.0):
        """Global (F(w_eff), #correct) with one all-reduce of two scalars."""
        buf, out = self.objective_parts_device(w, direction, alpha)
        (loss, ncorr), (_, wsq) = buf.tolist(), out.tolist()
        return loss + 0.5 * self.lam * wsq, int(round(ncorr))

    def gradient_and_objective_device(self, w):
        """Fused pass at w over the full data: (global gradient + lam w, global
        [loss, #correct], local [loss, ||w||^2]); None where the fused pass is
        not built (CSR / wide classes)."""
        fused = softmax.gradient_and_correct(self.local, w, 1.0, 0.0)
        if fused is None:
            return None
        G, out, corr = fused
        all_reduce_(G, self.group)
        _lib.call("snx_finish_hv", ptr(w), self.lam, G.numel(), ptr(G), None, None,
                  stream_handle())
        buf = torch.stack([out[0], corr[0].to(torch.float64)])
        all_reduce_(buf, self.group)
        return G, buf, out


class ShardedHessian:
    """Sampled Hessian over all ranks: local X_S^T(...) with lam = 0, one
    all-reduce, then + lam v and the CG dot partials (snx_finish_hv)."""

    _snx_device = True

    def __init__(self, view, x, lam, scale, group=None):
        self.op = softmax.HessianOperator(view, x, 0.0, scale=scale)
        self.lam = float(lam)
        self.scale = float(scale)
        self.dim = self.op.dim
        self.group = group

    def apply_into(self, v, out, dots=None, skip=None):
        self.op.apply_into(v, out, None, skip)
        all_reduce_(out, self.group)
        _lib.call("snx_finish_hv", ptr(v), self.lam, self.dim, ptr(out), ptr(dots), skip,
                  stream_handle())
        return out

    def apply(self, v):
        vv, as_t = vec_in(v, self.dim, "vector")
        out = torch.empty_like(vv)
        self.apply_into(vv, out)
        return vec_out(out, as_t)

    __call__ = apply


class ShardedOracle:
    """SubsampledOracle (sampling.py:72-96) across ranks."""

    _snx_device = True

    def __init__(self, sp, cfg, iteration):
        self.sp = sp
        n = sp.n_global
        self.s_g, self.s_h = draw_samples(cfg, n, iteration)  # same bits on every rank
        self._view_g = sp.local.take(local_indices(self.s_g, sp.row0, sp.row1))
        self._view_h = sp.local.take(local_indices(self.s_h, sp.row0, sp.row1))
        self.scale_g = n / len(self.s_g)
        self.scale_h = n / len(self.s_h)

    def gradient_device(self, w):
        g, _ = softmax.gradient_parts(self._view_g, w, self.scale_g, 0.0)
        all_reduce_(g, self.sp.group)
        _lib.call("snx_finish_hv", ptr(w), self.sp.lam, g.numel(), ptr(g), None, None,
                  stream_handle())
        return g

    def gradient(self, x):
        w, as_t = vec_in(x, self.sp.dim)
        return vec_out(self.gradient_device(w), as_t)

    def hessian_operator(self, x):
        w, _ = vec_in(x, self.sp.dim)
        return ShardedHessian(self._view_h, w, self.sp.lam, self.scale_h, self.sp.group)


def newton_solve_sharded(sp, cfg, x0=None, solver_name="newton"):
    """newton.py:115-140 on a row-sharded problem; every rank returns the same trace.

    One host synchronisation per outer iteration, as newton.newton_solve: the
    gradient (all-reduced), CG (one all-reduce per product), the slope and the
    first Armijo trial (fused with the gradient at the trial point when S_g is
    the full set) are enqueued before the host reads the scalars."""
    d = sp.dim
    x, as_t = vec_in(np.zeros(d) if x0 is None else x0, d, "initial point")
    x = x.clone()
    n = sp.n_global
    a0 = cfg.ls.alpha0
    full_g = (not cfg.samples.with_replacement
              and sample_size(cfg.samples.gradient_fraction, n) == n)
    cgws = CgWorkspace(d, cfg.cg.max_iters, x.device)
    t0 = time.perf_counter()
    f_cur, corr = sp.objective_and_correct(x)
    records = [RunRecord(solver_name, 0, 0.0, f_cur, corr / n, math.nan, 0.0, 0)]
    reason = "max-iters"
    g_next = None
    for k in range(cfg.max_outer_iters):
        oracle = ShardedOracle(sp, cfg.samples, k)
        g = g_next if g_next is not None else oracle.gradient_device(x)
        g_next = None
        gg = dot(g, g)
        hess = oracle.hessian_operator(x)
        enqueue_cg(hess, g, cfg.cg.theta, cfg.cg.max_iters, cgws)
        p = cgws.pb.clone()
        slope_t = dot(p, g)
        x_try = axpy(x, a0, p)
        fused = sp.gradient_and_objective_device(x_try) if full_g else None
        if fused is not None:
            g_try, buf, out = fused
        else:
            g_try = None
            buf, out = sp.objective_parts_device(x_try)
        h_gg, h_slope, h_buf, h_out, h_slot = download(gg, slope_t, buf, out,
                                                       cgws.slot(cfg.cg.max_iters))
        if math.sqrt(float(h_gg)) < cfg.epsilon:
            reason = "gradient-converged"
            break
        report = report_from(cgws, cfg.cg.max_iters, True, slot_values=h_slot.tolist())
        if report.iterations == 0 and report.converged:
            p.zero_()  # cg.py:61-62
        seen = {a0: (float(h_buf[0]) + 0.5 * sp.lam * float(h_out[1]), int(round(h_buf[1])))}

        def trial(a):
            if a not in seen:
                seen[a] = sp.objective_and_correct(x, p, a)
            return seen[a][0]

        try:
            alpha, _ = line_search(trial, f_cur, float(h_slope), cfg.ls)
        except LineSearchError:
            reason = "line-search-failure"
            break
        if alpha == a0:
            x = x_try
            g_next = g_try
        else:
            x = axpy(x, alpha, p)
        f_cur, corr = seen[alpha]
        records.append(RunRecord(solver_name, k + 1, time.perf_counter() - t0, f_cur, corr / n,
                                 math.nan, alpha, report.iterations))
    return SolveTrace(records, vec_out(x, as_t), reason)
