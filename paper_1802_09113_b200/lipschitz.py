"""Power-iteration estimate of the Lipschitz constant L of the gradient: the
largest eigenvalue of the unregularised Hessian at x = 0 -- the reference's
estimate_lipschitz (bench.py:116-138), the second consumer of the Hessian
product (it seeds the first-order learning-rate grid and the condition-number
estimate (L + lam) / lam).

Each iteration is one full-data snx_hess_apply (w = H v) plus snx_power_step
(Rayleigh quotient v.w, ||w||, v = w / ||w||, zero test) -- all enqueued on the
device; the host reads the estimate once at the end.  The start vector is the
reference's (POWER stream, rng.py:21), drawn on the host.
"""

import numpy as np
import torch

from . import _lib
from .device import as_device, ptr, stream_handle
from .errors import DataError
from .rng import POWER_STREAM, stream_rng
from .softmax import HessianOperator


def estimate_lipschitz(prob, iters=200, seed=0):
    """Rayleigh quotient of the final power iterate (bench.py:116-138)."""
    view = as_device(prob.dataset)
    if view.n_rows == 0:
        raise DataError("cannot estimate the Lipschitz constant of an empty dataset")
    d = view.dim
    dev = view.X.device
    op = HessianOperator(view, torch.zeros(d, dtype=torch.float64, device=dev), lam=0.0)
    v0 = stream_rng(seed, POWER_STREAM).standard_normal(d)
    v0 /= np.linalg.norm(v0)
    v = torch.from_numpy(v0).to(dev)
    w = torch.empty_like(v)
    state = torch.zeros(_lib.POWER_STATE, dtype=torch.float64, device=dev)
    zero_flag = ptr(state) + 2 * 8
    for _ in range(iters):
        op.apply_into(v, w, skip=zero_flag)
        _lib.call("snx_power_step", ptr(v), ptr(w), d, ptr(state), stream_handle())
    if iters <= 0:
        return 0.0
    rq, _, zero = state[:3].tolist()
    return 0.0 if zero != 0.0 else rq


__all__ = ["estimate_lipschitz"]
