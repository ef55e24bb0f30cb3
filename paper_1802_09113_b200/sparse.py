"""Sparse (CSR) datasets in HBM -- the reference's sparse DesignMatrix
(dataset.py:21-147: validated CSR, `take` row gather, `matmat` / `rmatmat`
products) for the paper's Newsgroups20-style data (cuSPARSE).

A `CsrDataset` keeps the rows twice: CSR (the logits pass, one warp per row)
and its transpose CSC (the X^T R pass, one warp per column), so every
reduction runs in a fixed order without atomics (csrc/snx_csr.cu).  The CSC
copy is made once on the host at upload (scipy's tocsc, part of ingest); a
row sample (a Hessian sample S_H, a gradient sample S_g, a test split) is
materialised on the device by snx_csr_gather, which also filters the CSC.

fp64 only (the parity path) and K = C - 1 <= 32 (Newsgroups20: C = 20).
"""

import numpy as np
import torch

from . import _lib
from .device import cuda_device, ptr, stream_handle, upload
from .errors import DataError, DimensionError


class CsrDataset:
    """CSR + CSC features (fp64) and int32 labels in HBM."""

    is_sparse = True
    code = _lib.F64
    dtype = "f64"

    def __init__(self, indptr, indices, data, colptr, rowidx, cdata, labels, n_classes, n_features,
                 host_indptr):
        if n_classes < 2:
            raise DataError(f"need at least 2 classes, got {n_classes}")
        if n_classes - 1 > 1 << 16:
            raise DataError(f"C = {n_classes} classes: too many for the sparse path")
        self.indptr, self.indices, self.data = indptr, indices, data
        self.colptr, self.rowidx, self.cdata = colptr, rowidx, cdata
        self.labels = labels
        self.n_classes = int(n_classes)
        self.n_features = int(n_features)
        self.host_indptr = host_indptr  # row lengths for sample capacities
        self._ws = None
        self._hess = {}
        self.rows = None

    # ------------------------------------------------------------ construction
    @classmethod
    def from_scipy(cls, mat, labels, n_classes):
        import scipy.sparse as sp

        dev = cuda_device()
        csr = sp.csr_array(mat, dtype=np.float64)
        n, p = csr.shape
        y = np.asarray(labels, dtype=np.int64)
        if len(y) != n:
            raise DimensionError(f"{len(y)} labels for {n} rows")
        if len(y) and (y.min() < 0 or y.max() >= n_classes):
            raise DataError(f"labels must lie in [0, {n_classes})")
        indptr = np.asarray(csr.indptr, dtype=np.int64)
        if indptr[0] != 0 or np.any(np.diff(indptr) < 0) or indptr[-1] != len(csr.data):
            raise DataError("malformed CSR row offsets")  # dataset.py:44-51
        csc = csr.tocsc()  # rows ascending within each column
        f64 = lambda a: upload(np.asarray(a, dtype=np.float64), dev)  # noqa: E731
        i32 = lambda a: upload(np.asarray(a, dtype=np.int32), dev)  # noqa: E731
        i64 = lambda a: upload(np.asarray(a, dtype=np.int64), dev)  # noqa: E731
        return cls(i64(indptr), i32(csr.indices), f64(csr.data), i64(csc.indptr), i32(csc.indices),
                   f64(csc.data), i32(y), n_classes, p, indptr)

    @property
    def host_labels(self):
        hl = getattr(self, "_host_labels", None)
        if hl is None:
            hl = self._host_labels = self.labels.cpu().numpy()
        return hl

    @classmethod
    def from_dataset(cls, ds):
        """From the reference's LabeledDataset with sparse features (duck-typed:
        features._mat / toarray, labels, n_classes)."""
        mat = getattr(ds.features, "_mat", None)
        if mat is None:
            import scipy.sparse as sp

            mat = sp.csr_array(ds.features.toarray())
        return cls.from_scipy(mat, ds.labels, ds.n_classes)

    # ------------------------------------------------------------ shape
    n_rows = property(lambda self: int(self.indptr.numel()) - 1)
    K = property(lambda self: self.n_classes - 1)
    dim = property(lambda self: self.K * self.n_features)
    nnz = property(lambda self: int(self.data.numel()))
    base = property(lambda self: self)
    X = property(lambda self: self.data)  # device of the dataset (HessianOperator uses .device)

    def materialized(self):
        return self

    # ------------------------------------------------------------ views
    def take(self, indices, _sorted=False):
        """Row gather (dataset.py:90-97); identity returns self (`_sorted`: see
        DeviceDataset.take)."""
        idx = np.asarray(indices, dtype=np.int64)
        n = self.n_rows
        if len(idx) == n and np.array_equal(idx, np.arange(n)):
            return self
        if len(idx) and (idx.min() < 0 or idx.max() >= n if not _sorted
                         else idx[0] < 0 or idx[-1] >= n):
            raise DimensionError("row index out of range")
        return CsrView(self, idx)

    def slice_rows(self, i0, i1):
        return self.take(np.arange(i0, i1))

    def sample_nnz(self, idx):
        ip = self.host_indptr
        return int((ip[idx + 1] - ip[idx]).sum()) if len(idx) else 0

    def gather(self, rows_dev, m, nnz, out=None):
        """(indptr, indices, data, colptr, rowidx, cdata) of rows `rows_dev` (device int64)."""
        dev = self.data.device
        if out is None:
            out = CsrSample(m, self.n_features, max(nnz, 1), dev)
        ws = self.workspace(self.n_rows)
        _lib.call("snx_csr_gather", ptr(self.indptr), ptr(self.indices), ptr(self.data),
                  ptr(self.colptr), ptr(self.rowidx), ptr(self.cdata), self.n_rows,
                  self.n_features, ptr(rows_dev), m, ptr(out.indptr), ptr(out.indices),
                  ptr(out.data), ptr(out.colptr), ptr(out.rowidx), ptr(out.cdata), ptr(ws),
                  ws.numel(), stream_handle())
        return out

    def hess_buffers(self, m, gathered):
        key = (m, gathered)
        hb = self._hess.get(key)
        if hb is None:
            hb = self._hess[key] = CsrHessBuffers(self, m, gathered)
        return hb

    # ------------------------------------------------------------ workspace
    def workspace(self, nrows):
        need = int(_lib.load().snx_csr_workspace_bytes(max(nrows, self.n_rows), self.n_features,
                                                       self.K))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.zeros(need, dtype=torch.uint8, device=self.data.device)
        return self._ws


class CsrSample:
    """Device CSR + CSC buffers of a row sample with room for `cap` entries."""

    def __init__(self, m, p, cap, dev):
        i64 = dict(dtype=torch.int64, device=dev)
        self.cap = cap
        self.indptr = torch.zeros(m + 1, **i64)
        self.colptr = torch.zeros(p + 1, **i64)
        self.indices = torch.empty(cap, dtype=torch.int32, device=dev)
        self.rowidx = torch.empty(cap, dtype=torch.int32, device=dev)
        self.data = torch.empty(cap, dtype=torch.float64, device=dev)
        self.cdata = torch.empty(cap, dtype=torch.float64, device=dev)


class CsrHessBuffers:
    """Sample buffers of the sparse Hessian operators of m rows (shared by the
    operators of one dataset and sample size, like device.HessBuffers, so the
    captured CG graph stays valid); capacity grows only if a sample with
    replacement needs more entries than the dataset holds (graphs dropped)."""

    xs_tc = None

    def __init__(self, base, m, gathered):
        dev = base.data.device
        self.base, self.m, self.gathered = base, m, gathered
        self.sample = CsrSample(m, base.n_features, max(base.nnz, 1), dev) if gathered else None
        self.h = torch.empty((max(m, 1), base.K), dtype=torch.float64, device=dev)
        self.owner = None
        self.graphs = {}

    def ensure(self, nnz):
        if self.sample is not None and nnz > self.sample.cap:
            self.sample = CsrSample(self.m, self.base.n_features, nnz, self.base.data.device)
            self.graphs = {}


class CsrView:
    """Rows `idx` of a CsrDataset; materialised (CSR + CSC of the rows) on first
    use by a full-data pass."""

    is_sparse = True
    code = _lib.F64
    dtype = "f64"

    def __init__(self, base, idx):
        self.base = base
        self.idx = idx
        self.rows = upload(idx, base.data.device)
        self._dense = None

    def materialized(self):
        if self._dense is None:
            b = self.base
            s = b.gather(self.rows, len(self.idx), b.sample_nnz(self.idx))
            lab = upload(b.host_labels[self.idx], b.data.device)
            self._dense = CsrDataset(s.indptr, s.indices, s.data, s.colptr, s.rowidx, s.cdata,
                                     lab, b.n_classes, b.n_features,
                                     np.concatenate([[0], np.cumsum(
                                         b.host_indptr[self.idx + 1] - b.host_indptr[self.idx])]))
        return self._dense

    n_rows = property(lambda self: len(self.idx))
    n_features = property(lambda self: self.base.n_features)
    n_classes = property(lambda self: self.base.n_classes)
    K = property(lambda self: self.base.K)
    dim = property(lambda self: self.base.dim)
    X = property(lambda self: self.base.data)
    labels = property(lambda self: self.materialized().labels)

    def workspace(self, nrows):
        return self.base.workspace(nrows)


# ------------------------------------------------------------------ passes
def objective_parts(view, w, direction=None, alpha=0.0, want_correct=False):
    ds = view.materialized()
    out = torch.empty(2, dtype=torch.float64, device=w.device)
    corr = torch.empty(1, dtype=torch.int64, device=w.device) if want_correct else None
    ws = ds.workspace(ds.n_rows)
    _lib.call("snx_csr_objective", ptr(ds.indptr), ptr(ds.indices), ptr(ds.data), ds.n_rows,
              ds.n_features, ds.K, ptr(ds.labels), ptr(w), ptr(direction), float(alpha),
              ptr(out), ptr(corr), ptr(ws), ws.numel(), stream_handle())
    return out, corr


def gradient_parts(view, w, scale, lam):
    ds = view.materialized()
    out = torch.empty(2, dtype=torch.float64, device=w.device)
    G = torch.empty_like(w)
    ws = ds.workspace(ds.n_rows)
    _lib.call("snx_csr_objective_grad", ptr(ds.indptr), ptr(ds.indices), ptr(ds.data),
              ptr(ds.colptr), ptr(ds.rowidx), ptr(ds.cdata), ds.n_rows, ds.n_features, ds.K,
              ptr(ds.labels), ptr(w), float(scale), float(lam), ptr(out), ptr(G), ptr(ws),
              ws.numel(), stream_handle())
    return G, out


def hess_prepare(op):
    """Gather the operator's sample (CSR + CSC) and its probabilities h."""
    view, hb = op.view, op._bufs
    base = view.base
    if hb.gathered:
        hb.ensure(base.sample_nnz(view.idx))
        base.gather(view.rows, view.n_rows, 0, out=hb.sample)
        src = hb.sample
    else:
        src = base
    ws = base.workspace(base.n_rows)
    _lib.call("snx_csr_hess_prepare", ptr(src.indptr), ptr(src.indices), ptr(src.data),
              view.n_rows, base.n_features, base.K, ptr(op._w), ptr(hb.h), ptr(ws), ws.numel(),
              stream_handle())


def hess_apply(op, v, out, dots=None, skip=None):
    view, hb = op.view, op._bufs
    base = view.base
    src = hb.sample if hb.gathered else base
    ws = base.workspace(base.n_rows)
    _lib.call("snx_csr_hess_apply", ptr(src.indptr), ptr(src.indices), ptr(src.data),
              ptr(src.colptr), ptr(src.rowidx), ptr(src.cdata), view.n_rows, base.n_features,
              base.K, ptr(hb.h), ptr(v), op.scale, op.lam, ptr(out), ptr(dots), skip, ptr(ws),
              ws.numel(), stream_handle())
    return out


__all__ = ["CsrDataset", "CsrView", "objective_parts", "gradient_parts"]
