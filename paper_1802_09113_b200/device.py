"""HBM-resident datasets, row views and d-vector plumbing.

A `DeviceDataset` is the B200 counterpart of the reference's LabeledDataset
(dataset.py:150-190): the feature matrix lives in HBM, row-major with a
16-byte aligned leading dimension, in the compute dtype ("f64": the 1e-10
parity path, "f32": the 1e-4 path); labels are int32.  `take(indices)` is the
row gather of dataset.py:90-97 -- it does not copy rows, it returns a view
holding the (sorted) indices, which the kernels gather through (the fused
gather-GEMM of the north star).  The identity selection returns the dataset
itself, as the reference does, so full-sample runs use the unsampled path.

torch owns the device memory; all arithmetic is done by libsnx kernels.
"""

import os
import weakref

import numpy as np
import torch

from . import _lib
from .errors import DataError, DimensionError

DTYPES = {"f64": (_lib.F64, torch.float64), "f32": (_lib.F32, torch.float32)}


def cuda_device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1802_09113_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_handle():
    """cudaStream_t of the current stream (the raw getter skips building a
    torch Stream object: ~0.5 instead of ~6 us per kernel-launching call)."""
    if _RAW_STREAM is not None:
        return _RAW_STREAM(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


def _out_of_range(idx, n):
    return bool(idx.min() < 0 or idx.max() >= n)


def ptr(t):
    return None if t is None else t.data_ptr()


def round_up(x, a):
    return (x + a - 1) // a * a


class DeviceDataset:
    """Features (n x p, padded to ld) + int32 labels in HBM."""

    def __init__(self, X, labels, n_classes, n_features, dtype="f64"):
        if dtype not in DTYPES:
            raise ValueError(f"dtype must be one of {sorted(DTYPES)}, got {dtype!r}")
        if n_classes < 2:
            raise DataError(f"need at least 2 classes, got {n_classes}")
        if dtype != "f64" and n_classes - 1 > 128:
            raise DataError(f"C = {n_classes} classes: f32 data supports C <= 129 (the wide "
                            "tensor-core path); fp64 data takes any C")
        self.X = X
        self.labels = labels
        self.n_classes = int(n_classes)
        self.n_features = int(n_features)
        self.dtype = dtype
        self.code = DTYPES[dtype][0]
        self.ld = int(X.shape[1])
        self._ws = None
        self._hess = {}   # m -> HessBuffers (sample buffers shared by operators)
        self.rows = None  # a dataset is its own identity view

    # ------------------------------------------------------------ construction
    @classmethod
    def from_numpy(cls, features, labels, n_classes, dtype="f64"):
        dev = cuda_device()
        A = np.ascontiguousarray(features, dtype=np.float64)
        if A.ndim != 2:
            raise DimensionError(f"feature matrix must be 2-D, got shape {A.shape}")
        y = np.asarray(labels, dtype=np.int64)
        n, p = A.shape
        if len(y) != n:
            raise DimensionError(f"{len(y)} labels for {n} rows")
        if n_classes < 2:
            raise DataError(f"need at least 2 classes, got {n_classes}")
        if len(y) and (y.min() < 0 or y.max() >= n_classes):
            raise DataError(f"labels must lie in [0, {n_classes})")
        code, tdtype = DTYPES.get(dtype, (None, None))
        if code is None:
            raise ValueError(f"dtype must be one of {sorted(DTYPES)}, got {dtype!r}")
        ld = max(4, round_up(p, 4))
        X = torch.empty((n, ld), dtype=tdtype, device=dev)
        if n:
            if code == _lib.F64 and ld == p:
                X.copy_(torch.from_numpy(A))
            else:
                stage = torch.from_numpy(A).to(dev)
                _lib.call("snx_pack_rows", code, ptr(stage), n, p, ptr(X), ld, stream_handle())
                del stage
        lab = torch.from_numpy(y.astype(np.int32)).to(dev)
        return cls(X, lab, n_classes, p, dtype)

    @classmethod
    def from_dataset(cls, ds, dtype="f64"):
        """From the reference's LabeledDataset (duck-typed: features.toarray(), labels,
        n_classes) or anything with the same fields."""
        feats = ds.features
        A = feats.toarray() if hasattr(feats, "toarray") else np.asarray(feats)
        return cls.from_numpy(A, ds.labels, ds.n_classes, dtype=dtype)

    # ------------------------------------------------------------ shape
    @property
    def n_rows(self):
        return int(self.X.shape[0])

    @property
    def K(self):
        return self.n_classes - 1

    @property
    def dim(self):
        return self.K * self.n_features

    @property
    def base(self):
        return self

    def materialized(self):
        return self

    # ------------------------------------------------------------ views
    def take(self, indices, _sorted=False):
        """Row gather (dataset.py:90-97, 180-185); identity returns self.
        `_sorted`: the indices are ascending (the sampler's sets): the range
        check reads the two ends only."""
        idx = np.asarray(indices, dtype=np.int64)
        n = self.n_rows
        if len(idx) == n and np.array_equal(idx, np.arange(n)):
            return self
        if len(idx) and (_out_of_range(idx, n) if not _sorted else idx[0] < 0 or idx[-1] >= n):
            raise DimensionError("row index out of range")
        return DeviceView(self, upload(idx, self.X.device), len(idx))

    def slice_rows(self, i0, i1):
        return self.take(np.arange(i0, i1))

    def hess_buffers(self, m, gathered):
        """Persistent sample buffers (X_S, h) for Hessian operators of m rows."""
        key = (m, gathered)
        hb = self._hess.get(key)
        if hb is None:
            hb = self._hess[key] = HessBuffers(self, m, gathered)
        return hb

    # ------------------------------------------------------------ tensor-core split
    def tc_split(self):
        """bf16 split X1 + X2 of the f32 rows (the wide-class objective / gradient
        passes read it); made once and cached."""
        split = getattr(self, "_tc_split", None)
        if split is None:
            ldb = int(_lib.load().snx_tc_ld(self.n_features))
            xs = torch.empty((2, max(self.n_rows, 1), ldb), dtype=torch.bfloat16,
                             device=self.X.device)
            _lib.call("snx_tc_split", ptr(self.X), self.ld, self.n_rows, self.n_features,
                      ptr(xs[0]), ptr(xs[1]), ldb, stream_handle())
            split = self._tc_split = (xs, ldb)
        return split

    # ------------------------------------------------------------ workspace
    def workspace(self, nrows):
        owner = getattr(self, "_ws_owner", None)
        if owner is not None:  # a materialised view shares its parent's workspace
            return owner.workspace(nrows)
        cache = self.__dict__.setdefault("_ws_need", {})
        need = cache.get(nrows)
        if need is None:
            need = cache[nrows] = _lib.workspace_bytes(self.code, nrows, self.n_features, self.K)
        if self._ws is None or self._ws.numel() < need:
            floor = _lib.workspace_bytes(self.code, self.n_rows, self.n_features, self.K)
            self._ws = torch.zeros(max(need, floor), dtype=torch.uint8, device=self.X.device)
        return self._ws


# f32 data with K <= 9 takes the one-pass kernel (rows widened to fp64); True
# sends it to the tcgen05 pair instead (A/B measurements: bench.py)
F32_TENSOR_CORES = os.environ.get("SNX_F32_TC") == "1"


class HessBuffers:
    """HBM buffers of one sampled Hessian (the sample's rows and h probabilities).

    Operators of the same dataset and sample size share them, so every outer
    iteration reuses the same addresses and the captured CUDA graph of the CG
    loop (cg.CgGraph) stays valid.  `owner` is the operator whose sample is
    currently prepared; any other operator re-prepares before use.

    K <= 9 (`fused`, fp64 or f32 data): the one-pass kernels read the sample in
    place through its row indices (a fixed-address copy in `rows`); h is fp64
    and nothing else is materialised (f32 rows are widened to fp64 in shared
    memory).  Otherwise the rows are gathered into `xs` (and, for f32, the bf16
    split X1 + X2 the tensor-core product reads)."""

    def __init__(self, base, m, gathered):
        dev = base.X.device
        mm = max(m, 1)
        self.fused = bool(_lib.load().snx_rowpass_fused(base.code, base.n_features, base.K)) \
            and not (base.code == _lib.F32 and F32_TENSOR_CORES)
        self.rows = None
        self.xs = None
        if self.fused:
            if gathered:
                self.rows = torch.empty(mm, dtype=torch.int64, device=dev)
        else:
            self.xs = torch.empty((mm, base.ld), dtype=base.X.dtype, device=dev) if gathered \
                else base.X
        self.h = torch.empty((mm, base.K), dtype=torch.float64 if self.fused else base.X.dtype,
                             device=dev)
        # f32: bf16 split X1 + X2 of the sample rows for the tensor-core product
        self.xs_tc = None
        if base.code == _lib.F32 and not self.fused:
            self.ldb = int(_lib.load().snx_tc_ld(base.n_features))
            rows = mm if gathered else max(base.X.shape[0], 1)
            self.xs_tc = torch.empty((2, rows, self.ldb), dtype=torch.bfloat16, device=dev)
        self.owner = None
        self.graphs = {}


class DeviceView:
    """Rows `rows` (sorted int64 device indices) of a DeviceDataset.

    Kernels stream contiguous rows (TMA tiles), so a view used by a full pass
    is materialised once (snx_gather_rows) and cached; the Hessian operator
    gathers its sample itself (snx_hess_prepare)."""

    def __init__(self, base, rows, n_rows):
        self.base = base
        self.rows = rows
        self._n = int(n_rows)
        self._dense = None

    def materialized(self):
        if self._dense is None:
            b = self.base
            X = torch.empty((self._n, b.ld), dtype=b.X.dtype, device=b.X.device)
            lab = torch.empty(self._n, dtype=torch.int32, device=b.X.device)
            _lib.call("snx_gather_rows", b.code, ptr(b.X), b.ld, ptr(b.labels), ptr(self.rows),
                      self._n, ptr(X), b.ld, ptr(lab), stream_handle())
            self._dense = DeviceDataset(X, lab, b.n_classes, b.n_features, b.dtype)
            self._dense._ws = b._ws
            self._dense._ws_owner = b
        return self._dense

    def take(self, indices, _sorted=False):
        """Rows `indices` of this view (a view of the base's rows[indices]):
        sampling from a train split works as on the reference's materialised
        LabeledDataset (dataset.py:180-185)."""
        idx = np.asarray(indices, dtype=np.int64)
        n = self._n
        if len(idx) == n and np.array_equal(idx, np.arange(n)):
            return self
        if len(idx) and (_out_of_range(idx, n) if not _sorted else idx[0] < 0 or idx[-1] >= n):
            raise DimensionError("row index out of range")
        return DeviceView(self.base, self.rows[upload(idx, self.rows.device)], len(idx))

    def slice_rows(self, i0, i1):
        return self.take(np.arange(i0, i1))

    n_features = property(lambda self: self.base.n_features)
    n_classes = property(lambda self: self.base.n_classes)
    K = property(lambda self: self.base.K)
    dim = property(lambda self: self.base.dim)
    dtype = property(lambda self: self.base.dtype)
    code = property(lambda self: self.base.code)
    X = property(lambda self: self.base.X)
    ld = property(lambda self: self.base.ld)
    labels = property(lambda self: self.base.labels)

    @property
    def n_rows(self):
        return self._n

    def workspace(self, nrows):
        return self.base.workspace(nrows)


# Reference-dataset objects are uploaded once and cached (keyed by identity).
_CACHE = {}


def as_device(ds, dtype="f64"):
    if isinstance(ds, (DeviceDataset, DeviceView)) or getattr(ds, "is_sparse", False) is True:
        return ds
    key = (id(ds), dtype)
    hit = _CACHE.get(key)
    if hit is not None and hit[0]() is ds:
        return hit[1]
    if getattr(getattr(ds, "features", None), "is_sparse", False):  # reference CSR storage
        from .sparse import CsrDataset

        dev = CsrDataset.from_dataset(ds)
    else:
        dev = DeviceDataset.from_dataset(ds, dtype=dtype)
    try:
        ref = weakref.ref(ds, lambda _r, k=key: _CACHE.pop(k, None))
    except TypeError:  # not weak-referenceable: keep a strong reference
        ref = (lambda obj: (lambda: obj))(ds)
    _CACHE[key] = (ref, dev)
    return dev


def upload(a, device=None):
    """numpy -> device, asynchronous on the current stream (the host goes on
    enqueueing work instead of waiting for the GPU to drain).  Up to 4 MB the
    copy goes straight from the pageable array: the driver stages it before
    returning (the caller may reuse the array at once; no device or stream
    synchronisation), measured cheaper than a pinned allocation per call
    (`tools/upload_ab.py`); larger arrays go through torch's pinned host cache."""
    a = np.ascontiguousarray(a)
    dev = device or cuda_device()
    if a.nbytes <= 1 << 22:
        return torch.from_numpy(a).to(dev, non_blocking=True)
    return torch.from_numpy(a).pin_memory().to(dev, non_blocking=True)


def download(*ts):
    """Device tensors -> numpy arrays: asynchronous copies into pinned buffers and
    ONE stream synchronisation for all of them."""
    outs = []
    for t in ts:
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        outs.append(h)
    torch.cuda.current_stream().synchronize()
    return [h.numpy() for h in outs]


class AsyncRead:
    """Device tensors -> numpy without a stream synchronisation: copies into
    pinned buffers are enqueued now, `wait()` blocks on an event recorded after
    them (work enqueued later keeps the GPU busy meanwhile)."""

    def __init__(self, *ts):
        self.bufs = []
        for t in ts:
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t, non_blocking=True)
            self.bufs.append(h)
        self.event = torch.cuda.Event()
        self.event.record()

    def wait(self):
        self.event.synchronize()
        return [h.numpy() for h in self.bufs]


def vec_in(x, d, what="weight vector"):
    """User vector -> (contiguous fp64 CUDA tensor of length d, caller_used_torch)."""
    if isinstance(x, torch.Tensor):
        if x.dim() != 1 or x.numel() != d:
            raise DimensionError(f"expected {what} of length {d}, got {tuple(x.shape)}")
        return x.to(device=cuda_device(), dtype=torch.float64).contiguous(), True
    a = np.asarray(x, dtype=np.float64)
    if a.shape != (d,):
        raise DimensionError(f"expected {what} of length {d}, got {a.shape}")
    return upload(a), False


def vec_out(t, as_torch):
    return t if as_torch else download(t)[0]


def dot(x, y):
    """Fixed-order device dot product (np.dot); returns a 0-d device tensor view."""
    out = torch.empty(1 + _lib.DOT_BLOCKS, dtype=torch.float64, device=x.device)
    _lib.call("snx_dot", ptr(x), ptr(y), x.numel(), ptr(out), stream_handle())
    return out[0]


def axpy(x, alpha, p, out=None):
    """x + alpha * p with numpy rounding (newton.py:97)."""
    out = torch.empty_like(x) if out is None else out
    _lib.call("snx_axpy", ptr(x), ptr(p), float(alpha), x.numel(), ptr(out), stream_handle())
    return out


def axpby(a, x, b, y, out=None):
    out = torch.empty_like(x) if out is None else out
    _lib.call("snx_axpby", float(a), ptr(x), float(b), ptr(y), x.numel(), ptr(out),
              stream_handle())
    return out
