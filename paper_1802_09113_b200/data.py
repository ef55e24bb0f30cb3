"""Dataset preparation on the device: normalize_columns and train_test_split
(the reference's dataset.py:314-342), so real data prepared the reference's
way feeds the GPU path without a host fp64 round trip.

normalize_columns -> snx_column_norms + snx_scale_columns (csrc/snx_data.cu);
train_test_split draws the reference's permutation on the host (the SPLIT
stream, rng.py:19) -- the row sets are bit-identical -- and returns device
row views.
"""

import numpy as np
import torch

from . import _lib
from .device import DeviceDataset, DeviceView, as_device, ptr, stream_handle
from .errors import DataError
from .rng import SPLIT_STREAM, stream_rng


def _csr_norms(base):
    p = base.n_features
    norms = torch.empty(max(p, 1), dtype=torch.float64, device=base.data.device)
    scale = torch.empty_like(norms)
    _lib.call("snx_csr_column_norms", ptr(base.colptr), ptr(base.cdata), p, ptr(norms),
              ptr(scale), stream_handle())
    return norms[:p], scale[:p]


def column_norms(ds):
    """Device fp64 Euclidean norms of the p feature columns (dataset.py:103-107)."""
    view = as_device(ds)
    if getattr(view, "is_sparse", False):
        return _csr_norms(view.materialized())
    base = view.materialized() if isinstance(view, DeviceView) else view
    p = base.n_features
    norms = torch.empty(max(p, 1), dtype=torch.float64, device=base.X.device)
    scale = torch.empty_like(norms)
    nbytes = int(_lib.load().snx_colnorm_workspace_bytes(p))
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=base.X.device)
    _lib.call("snx_column_norms", base.code, ptr(base.X), base.ld, base.n_rows, p, ptr(norms),
              ptr(scale), ptr(scratch), nbytes, stream_handle())
    return norms[:p], scale[:p]


def normalize_columns(ds):
    """Scale every column with nonzero norm to unit Euclidean norm; zero columns
    are left untouched (dataset.py:314-324).  Returns a new DeviceDataset; the
    input is not modified (inputs are immutable)."""
    view = as_device(ds)
    if getattr(view, "is_sparse", False):  # CSR: scale the stored values of both copies
        from .sparse import CsrDataset

        b = view.materialized()
        _, scale = _csr_norms(b)
        data, cdata = torch.empty_like(b.data), torch.empty_like(b.cdata)
        scratch = torch.empty(max(b.nnz, 1), dtype=torch.int32, device=b.data.device)
        _lib.call("snx_csr_scale_columns", ptr(b.indices), ptr(b.data), ptr(b.colptr),
                  ptr(b.cdata), b.nnz, b.n_features, ptr(scale), ptr(data), ptr(cdata),
                  ptr(scratch), stream_handle())
        return CsrDataset(b.indptr.clone(), b.indices.clone(), data, b.colptr.clone(),
                          b.rowidx.clone(), cdata, b.labels.clone(), b.n_classes, b.n_features,
                          b.host_indptr.copy())
    base = view.materialized() if isinstance(view, DeviceView) else view
    _, scale = column_norms(base)
    Y = torch.empty_like(base.X)
    _lib.call("snx_scale_columns", base.code, ptr(base.X), base.ld, base.n_rows,
              base.n_features, base.ld, ptr(scale), ptr(Y), base.ld, stream_handle())
    return DeviceDataset(Y, base.labels.clone(), base.n_classes, base.n_features, base.dtype)


def train_test_split(ds, train_fraction, seed):
    """Disjoint row partition of sizes (ceil(f*n), n - ceil(f*n)); rows keep their
    relative order (dataset.py:327-342).  Returns two device row views."""
    if not 0.0 < train_fraction < 1.0:
        raise DataError(f"train_fraction must be in (0, 1), got {train_fraction}")
    view = as_device(ds)
    n = view.n_rows
    if n < 2:
        raise DataError(f"need at least 2 rows to split, got {n}")
    n_train = int(np.ceil(train_fraction * n))
    perm = stream_rng(seed, SPLIT_STREAM).permutation(n)
    train_idx = np.sort(perm[:n_train])
    test_idx = np.sort(perm[n_train:])
    if getattr(view, "rows", None) is not None and view.base is not view:  # a row view
        rows = view.rows.cpu().numpy()
        return view.base.take(rows[train_idx]), view.base.take(rows[test_idx])
    return view.take(train_idx), view.take(test_idx)


__all__ = ["column_norms", "normalize_columns", "train_test_split"]
