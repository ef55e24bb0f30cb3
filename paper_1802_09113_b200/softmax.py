"""L2-regularised softmax cross-entropy on the GPU: objective, gradient and the
matrix-free sub-sampled Hessian operator.

Same names, argument meaning, layouts and exceptions as the reference's
softmax.py (file:line cited per function); the arithmetic runs in libsnx:

  objective / data_objective   -> snx_objective        (softmax.py:125-141)
  gradient  / data_gradient    -> snx_objective_grad   (softmax.py:144-169)
  HessianOperator.__init__     -> snx_hess_prepare     (softmax.py:181-195)
  HessianOperator.apply        -> snx_hess_apply       (softmax.py:197-212)
  accuracy                     -> snx_objective(correct_out)  (softmax.py:243-247)

Vectors may be numpy arrays (results come back as numpy, the reference's
contract) or CUDA torch tensors (results stay on the device).
"""

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, sparse
from .device import DeviceDataset, DeviceView, as_device, ptr, stream_handle, vec_in, vec_out
from .errors import DataError, DimensionError

BLOCK_ROWS = 8192  # accepted for API parity (softmax.py:25); kernels tile rows themselves
_UNFUSED = os.environ.get("SNX_CG_UNFUSED") == "1"  # A/B: unfused product + CG update


@dataclass(frozen=True)
class SoftmaxProblem:
    """A labeled dataset together with the regularisation coefficient (softmax.py:28-41)."""

    dataset: object
    lam: float

    def __post_init__(self):
        if self.lam < 0:
            raise DataError(f"regularization coefficient must be >= 0, got {self.lam}")

    @property
    def dim(self):
        return (self.dataset.n_classes - 1) * self.dataset.n_features


def zero_weights(p, n_classes):
    return np.zeros((n_classes - 1) * p, dtype=np.float64)


def weights_as_matrix(x, p, n_classes):
    """softmax.py:62-70: flat class-major x viewed as the p-by-(C-1) matrix."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape != ((n_classes - 1) * p,):
        raise DimensionError(
            f"weight vector must have length {(n_classes - 1) * p}, got {x.shape}")
    return x.reshape((p, n_classes - 1), order="F")


def matrix_as_weights(X):
    return np.asarray(X, dtype=np.float64).ravel(order="F")


def _view(ds):
    return as_device(ds)


def _args(ds):
    """Common leading ABI arguments for a contiguous (materialised) dataset."""
    return (ds.code, ptr(ds.X), ds.ld, ds.n_rows, ds.n_features, ds.K)


def _ws(view):
    ws = view.workspace(view.n_rows)
    return ptr(ws), ws.numel()


def _wide(view):
    """f32 data with more than 16 free classes: the tensor-core passes."""
    return view.code == _lib.F32 and view.K > 16


def _wide64(view):
    """fp64 data with more than 16 free classes: library DGEMMs + row kernels
    (csrc/snx_wide64.cu)."""
    return view.code == _lib.F64 and view.K > 16


_ZROWS = 32768  # rows per logits chunk of the wide fp64 passes (Z: ZROWS x K doubles)


def _wscratch(owner, n, p, K, device):
    """(scratch tensor, zrows) of a wide fp64 call over n rows, cached on `owner`
    (a dataset or the shared Hessian buffers: fixed addresses for graph replays)."""
    zr = min(max(int(n), 1), _ZROWS)
    need = int(_lib.load().snx_wide_scratch_doubles(int(n), p, K, zr))
    buf = getattr(owner, "_wide_scratch", None)
    if buf is None or buf.numel() < need:
        buf = torch.empty(need, dtype=torch.float64, device=device)
        owner._wide_scratch = buf
    return buf, zr


def objective_parts(view, w, direction=None, alpha=0.0, want_correct=False):
    """Device [data loss, ||w_eff||^2] (+ correct count) at w_eff = w + alpha*direction."""
    if getattr(view, "is_sparse", False):
        return sparse.objective_parts(view, w, direction, alpha, want_correct)
    view = view.materialized()
    out = torch.empty(2, dtype=torch.float64, device=w.device)
    corr = torch.empty(1, dtype=torch.int64, device=w.device) if want_correct else None
    if _wide(view):
        xs, ldb = view.tc_split()
        _lib.call("snx_objective_tc", ptr(xs[0]), ptr(xs[1]), ldb, view.n_rows,
                  view.n_features, view.K, ptr(view.labels), ptr(w), ptr(direction),
                  float(alpha), ptr(out), ptr(corr), *_ws(view), stream_handle())
        return out, corr
    if _wide64(view):
        sc, zr = _wscratch(view, view.n_rows, view.n_features, view.K, w.device)
        _lib.call("snx_wide_objective", ptr(view.X), view.ld, view.n_rows, view.n_features,
                  view.K, ptr(view.labels), ptr(w), ptr(direction), float(alpha), ptr(out),
                  ptr(corr), ptr(sc), zr, stream_handle())
        return out, corr
    _lib.call("snx_objective", *_args(view), ptr(view.labels), ptr(w), ptr(direction),
              float(alpha), ptr(out), ptr(corr), *_ws(view), stream_handle())
    return out, corr


def gradient_parts(view, w, scale, lam):
    """Device (G = scale * data_gradient + lam * w, [data loss, ||w||^2])."""
    if getattr(view, "is_sparse", False):
        return sparse.gradient_parts(view, w, scale, lam)
    view = view.materialized()
    out = torch.empty(2, dtype=torch.float64, device=w.device)
    G = torch.empty_like(w)
    if _wide(view):
        xs, ldb = view.tc_split()
        _lib.call("snx_objective_grad_tc", ptr(xs[0]), ptr(xs[1]), ldb, view.n_rows,
                  view.n_features, view.K, ptr(view.labels), ptr(w), float(scale), float(lam),
                  ptr(out), ptr(G), *_ws(view), stream_handle())
        return G, out
    if _wide64(view):
        sc, zr = _wscratch(view, view.n_rows, view.n_features, view.K, w.device)
        _lib.call("snx_wide_objective_grad", ptr(view.X), view.ld, view.n_rows,
                  view.n_features, view.K, ptr(view.labels), ptr(w), float(scale), float(lam),
                  ptr(out), ptr(G), ptr(sc), zr, stream_handle())
        return G, out
    _lib.call("snx_objective_grad", *_args(view), ptr(view.labels), ptr(w), float(scale),
              float(lam), ptr(out), ptr(G), *_ws(view), stream_handle())
    return G, out


def gradient_and_correct(view, w, scale, lam):
    """One pass: (G, [data loss, ||w||^2], correct count) -- snx_objective_grad_acc.
    None where that fused pass is not built (CSR / wide-class data): the caller
    evaluates the objective and the gradient separately."""
    if getattr(view, "is_sparse", False):
        return None
    view = view.materialized()
    if _wide(view) or _wide64(view):
        return None
    out = torch.empty(2, dtype=torch.float64, device=w.device)
    corr = torch.empty(1, dtype=torch.int64, device=w.device)
    G = torch.empty_like(w)
    _lib.call("snx_objective_grad_acc", *_args(view), ptr(view.labels), ptr(w), float(scale),
              float(lam), ptr(out), ptr(corr), ptr(G), *_ws(view), stream_handle())
    return G, out, corr


def data_objective(ds, x):
    """softmax.py:125-135: sum_i (maxPart_i + logPart_i - linearPart_i)."""
    view = _view(ds)
    w, _ = vec_in(x, view.dim)
    out, _ = objective_parts(view, w)
    return float(out[0])


def objective(prob, x):
    """softmax.py:138-141: data loss + (lam/2) ||x||^2."""
    view = _view(prob.dataset)
    w, _ = vec_in(x, view.dim, "weight vector")
    loss, wsq = objective_parts(view, w)[0].tolist()
    return loss + 0.5 * prob.lam * wsq


def data_gradient(ds, x):
    """softmax.py:144-163: vec(A^T (E/alpha - onehot))."""
    view = _view(ds)
    w, as_t = vec_in(x, view.dim)
    G, _ = gradient_parts(view, w, 1.0, 0.0)
    return vec_out(G, as_t)


def gradient(prob, x):
    """softmax.py:166-169: data gradient + lam x."""
    view = _view(prob.dataset)
    w, as_t = vec_in(x, view.dim)
    G, _ = gradient_parts(view, w, 1.0, prob.lam)
    return vec_out(G, as_t)


class HessianOperator:
    """v -> scale * H_data(x) v + lam * v over the rows of `ds` (softmax.py:172-212).

    The per-row softmax probabilities h(a_i, x_c) are computed once at
    construction (snx_hess_prepare) and kept in HBM; each `apply` costs one
    fused pass of two feature products (snx_hess_apply).
    """

    _snx_device = True

    def __init__(self, ds, x, lam, scale=1.0, block_rows=BLOCK_ROWS):
        view = _view(ds)
        w, from_torch = vec_in(x, view.dim)
        self.view = view
        self.ds = ds
        self.lam = float(lam)
        self.scale = float(scale)
        self.block_rows = block_rows
        self.p, self.C = view.n_features, view.n_classes
        self.dim = view.dim
        self._w = w.clone() if from_torch else w  # numpy input: w is already a private copy
        self._bufs = view.base.hess_buffers(view.n_rows, view.rows is not None)
        self._prepare()

    def _prepare(self):
        """Prepare this operator's sample and probabilities in the shared buffers."""
        view, base, hb = self.view, self.view.base, self._bufs
        if getattr(base, "is_sparse", False):  # CSR data (csrc/snx_csr.cu)
            sparse.hess_prepare(self)
        elif getattr(hb, "fused", False):  # fp64, K <= 9: gather fused into the one-pass kernel
            rows = None
            if view.rows is not None:
                hb.rows[:view.n_rows].copy_(view.rows)  # fixed address: graph replays
                rows = hb.rows
            _lib.call("snx_hess_prepare", base.code, ptr(base.X), base.ld, ptr(rows),
                      view.n_rows, view.n_features, view.K, ptr(self._w), None, base.ld,
                      ptr(hb.h), *_ws(view), stream_handle())
        elif _wide64(base):  # fp64, K > 16: library DGEMMs + row kernels
            sc, zr = _wscratch(hb, view.n_rows, self.p, view.K, base.X.device)
            _lib.call("snx_wide_hess_prepare", ptr(base.X), base.ld, ptr(view.rows), view.n_rows,
                      self.p, view.K, ptr(self._w), ptr(hb.xs), base.ld, ptr(hb.h), ptr(sc), zr,
                      stream_handle())
        elif hb.xs_tc is not None:  # f32: tensor-core product (csrc/snx_tc.cu)
            _lib.call("snx_hess_prepare_tc", ptr(base.X), base.ld, ptr(view.rows), view.n_rows,
                      view.n_features, view.K, ptr(self._w), ptr(hb.xs), base.ld, ptr(hb.h),
                      ptr(hb.xs_tc[0]), ptr(hb.xs_tc[1]), hb.ldb, *_ws(view), stream_handle())
        else:
            _lib.call("snx_hess_prepare", base.code, ptr(base.X), base.ld, ptr(view.rows),
                      view.n_rows, view.n_features, view.K, ptr(self._w), ptr(hb.xs), base.ld,
                      ptr(hb.h), *_ws(view), stream_handle())
        hb.owner = self

    @property
    def _h(self):
        if self._bufs.owner is not self:
            self._prepare()
        return self._bufs.h

    def apply_into(self, v, out, dots=None, skip=None):
        """Device-only apply: out = H v; optional CG dot partials and skip flag."""
        if self._bufs.owner is not self:
            self._prepare()
        base, hb = self.view.base, self._bufs
        if getattr(base, "is_sparse", False):
            return sparse.hess_apply(self, v, out, dots, skip)
        if getattr(hb, "fused", False):
            rows = hb.rows if self.view.rows is not None else None
            _lib.call("snx_hess_apply_rows", base.code, ptr(base.X), base.ld, ptr(rows),
                      self.view.n_rows, self.p, self.view.K, ptr(hb.h), ptr(v), self.scale,
                      self.lam, ptr(out), ptr(dots), skip, *_ws(self.view), stream_handle())
        elif _wide64(base):
            sc, zr = _wscratch(hb, self.view.n_rows, self.p, self.view.K, v.device)
            _lib.call("snx_wide_hess_apply", ptr(hb.xs), base.ld, self.view.n_rows, self.p,
                      self.view.K, ptr(hb.h), ptr(v), self.scale, self.lam, ptr(out), ptr(dots),
                      skip, ptr(sc), zr, stream_handle())
        elif hb.xs_tc is not None:
            _lib.call("snx_hess_apply_tc", ptr(hb.xs_tc[0]), ptr(hb.xs_tc[1]), hb.ldb,
                      self.view.n_rows, self.p, self.view.K, ptr(hb.h), ptr(v), self.scale,
                      self.lam, ptr(out), ptr(dots), skip, *_ws(self.view), stream_handle())
        else:
            _lib.call("snx_hess_apply", base.code, ptr(hb.xs), base.ld, self.view.n_rows,
                      self.p, self.view.K, ptr(hb.h), ptr(v), self.scale, self.lam, ptr(out),
                      ptr(dots), skip, *_ws(self.view), stream_handle())
        return out

    def apply_cg_into(self, t, T, ws):
        """CG iteration t on this operator with the product's finalize fused into
        the CG update (snx_hess_apply_cg_rows; fp64, K <= 9).  False: the caller
        runs apply_into + snx_cg_update.  SNX_CG_UNFUSED=1 forces the latter."""
        hb, view = self._bufs, self.view
        if not getattr(hb, "fused", False) or view.n_rows == 0 or _UNFUSED:
            return False
        if hb.owner is not self:
            self._prepare()
        base = view.base
        rows = hb.rows if view.rows is not None else None
        _lib.call("snx_hess_apply_cg_rows", base.code, ptr(base.X), base.ld, ptr(rows),
                  view.n_rows, self.p, view.K, ptr(hb.h), self.scale, self.lam, t, T,
                  ptr(ws.r), ptr(ws.s), ptr(ws.p), ptr(ws.pb), ptr(ws.Hs), ptr(ws.state),
                  *_ws(view), stream_handle())
        return True

    def apply(self, v):
        if isinstance(v, torch.Tensor) or np.asarray(v).shape == (self.dim,):
            vv, as_t = vec_in(v, self.dim, "vector")
        else:
            raise DimensionError(
                f"expected vector of length {self.dim}, got {np.asarray(v).shape}")
        out = torch.empty_like(vv)
        self.apply_into(vv, out)
        return vec_out(out, as_t)

    __call__ = apply


def hess_vec(prob, x, v):
    """softmax.py:215-221: one-shot operator + apply."""
    return HessianOperator(prob.dataset, x, prob.lam).apply(v)


@dataclass
class RowStats:
    """Per-row pieces of the stabilised loss (softmax.py:43-56): max_part M_i,
    sum_exp_part sum_c exp(z_ic - M_i), linear_part z_{i,b_i} (0 for the
    reference class).  numpy arrays when the weights came as numpy."""

    max_part: object
    sum_exp_part: object
    linear_part: object


def _probs_pass(ds, x, probs=False, pred=False, stats=False):
    """One device row pass (snx_class_probabilities / its CSR twin)."""
    view = _view(ds).materialized()
    w, as_t = vec_in(x, view.dim)
    n, C = view.n_rows, view.n_classes
    dev = w.device
    P = torch.empty((n, C), dtype=torch.float64, device=dev) if probs else None
    Y = torch.empty(n, dtype=torch.int32, device=dev) if pred else None
    S = torch.empty((n, 3), dtype=torch.float64, device=dev) if stats else None
    if n:
        if getattr(view, "is_sparse", False):
            ws = view.workspace(n)
            _lib.call("snx_csr_class_probabilities", ptr(view.indptr), ptr(view.indices),
                      ptr(view.data), n, view.n_features, view.K, ptr(view.labels), ptr(w),
                      ptr(P), ptr(Y), ptr(S), ptr(ws), ws.numel(), stream_handle())
        elif _wide(view):  # f32, K > 16: row chunks widened to fp64, the fp64 path
            zr = min(max(n, 1), 4096)
            need = int(_lib.load().snx_wide_f32_scratch_doubles(n, view.n_features, view.K, zr))
            sc = getattr(view, "_wide_scratch", None)
            if sc is None or sc.numel() < need:
                sc = view._wide_scratch = torch.empty(need, dtype=torch.float64, device=dev)
            _lib.call("snx_wide_class_probabilities_f32", ptr(view.X), view.ld, n,
                      view.n_features, view.K, ptr(view.labels), ptr(w), ptr(P), ptr(Y), ptr(S),
                      ptr(sc), zr, stream_handle())
        elif _wide64(view):
            sc, zr = _wscratch(view, n, view.n_features, view.K, dev)
            _lib.call("snx_wide_class_probabilities", ptr(view.X), view.ld, n, view.n_features,
                      view.K, ptr(view.labels), ptr(w), ptr(P), ptr(Y), ptr(S), ptr(sc), zr,
                      stream_handle())
        else:
            _lib.call("snx_class_probabilities", *_args(view), ptr(view.labels), ptr(w), ptr(P),
                      ptr(Y), ptr(S), *_ws(view), stream_handle())
    return P, Y, S, as_t


def class_probabilities(ds, x):
    """softmax.py:224-235: n-by-C probabilities, reference class last."""
    P, _, _, as_t = _probs_pass(ds, x, probs=True)
    return vec_out(P, as_t)


def predict(ds, x):
    """softmax.py:238-240: most probable class per row, ties to the lowest index."""
    _, Y, _, as_t = _probs_pass(ds, x, pred=True)
    return Y.long() if as_t else vec_out(Y, False).astype(np.int64)


def row_stats(ds, x):
    """softmax.py:107-122: RowStats for every row of ds at weights x."""
    _, _, S, as_t = _probs_pass(ds, x, stats=True)
    if as_t:
        return RowStats(S[:, 0], S[:, 1], S[:, 2])
    h = vec_out(S, False)
    return RowStats(h[:, 0].copy(), h[:, 1].copy(), h[:, 2].copy())


def correct_count(ds, x):
    """Device count of rows whose most probable class equals the label."""
    view = _view(ds)
    w, _ = vec_in(x, view.dim)
    _, corr = objective_parts(view, w, want_correct=True)
    return corr


def accuracy(ds, x):
    """softmax.py:243-247: fraction of rows predicted correctly (ties -> lowest class)."""
    view = _view(ds)
    if view.n_rows == 0:
        raise DataError("accuracy is undefined on an empty dataset")
    return float(correct_count(view, x)) / view.n_rows


__all__ = [
    "BLOCK_ROWS", "SoftmaxProblem", "zero_weights", "weights_as_matrix", "matrix_as_weights",
    "data_objective", "objective", "data_gradient", "gradient", "HessianOperator", "hess_vec",
    "accuracy", "correct_count", "objective_parts", "gradient_parts", "DeviceDataset",
    "DeviceView", "RowStats", "row_stats", "class_probabilities", "predict",
]
