"""Dataset text ingest straight to HBM: LIBSVM / svmlight and CSV (the reference's
load_libsvm / load_csv, dataset.py:242-311), so real datasets (covertype,
Newsgroups20, ... -- PAPER.md:700-702) feed the device path.

The LIBSVM text is parsed by native code (snx_libsvm_scan / snx_libsvm_fetch,
csrc/snx_io.cu) into CSR arrays; labels are remapped to 0..C-1 by sorted raw
value (dataset.py:200-213, the highest raw label becomes the reference class)
and the storage is picked as the reference does (dataset.py:216-226: CSR
unless more than 25 % of the entries are nonzero, or as requested), then the
arrays are uploaded: a sparse.CsrDataset or a dense DeviceDataset.
"""

import ctypes
import re

import numpy as np

from . import _lib
from .device import DeviceDataset
from .errors import DataError, ParseError
from .sparse import CsrDataset

DENSE_DENSITY_THRESHOLD = 0.25  # dataset.py:18


def remap_labels(raw, n_classes):
    """Raw label values -> 0..K-1 by sorted order (dataset.py:200-213)."""
    raw = np.asarray(raw, dtype=np.float64)
    distinct = np.unique(raw)
    if len(distinct) > n_classes:
        raise DataError(
            f"found {len(distinct)} distinct labels but only {n_classes} classes declared")
    return np.searchsorted(distinct, raw).astype(np.int64)


def picks_dense(csr, storage):
    """The storage choice of dataset.py:216-226 (True: dense rows)."""
    if storage not in ("auto", "dense", "sparse"):
        raise ValueError(f"storage must be auto|dense|sparse, got {storage!r}")
    n, p = csr.shape
    density = csr.nnz / (n * p) if n * p else 0.0
    return storage == "dense" or (storage == "auto" and density > DENSE_DENSITY_THRESHOLD)


def parse_libsvm(path, n_classes, n_features=None):
    """Host part of load_libsvm: (scipy CSR, 0-based labels)."""
    import scipy.sparse as sp

    raw, indptr, indices, data, max_index = read_libsvm(path)
    p = max_index if n_features is None else int(n_features)
    if n_features is not None and max_index > n_features:
        raise DataError(f"file uses feature index {max_index} > declared {n_features}")
    csr = sp.csr_array((data, indices, indptr), shape=(len(raw), p))
    return csr, remap_labels(raw, n_classes)


def _to_device(csr, labels, n_classes, storage, dtype):
    """Storage choice of dataset.py:216-226, then upload."""
    if picks_dense(csr, storage) or dtype != "f64":
        return DeviceDataset.from_numpy(csr.toarray(), labels, n_classes, dtype=dtype)
    return CsrDataset.from_scipy(csr, labels, n_classes)


def read_libsvm(path):
    """(raw labels, indptr, indices, data, max_index) parsed by libsnx."""
    lib = _lib.load()
    n, nnz, mx = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    bpath = str(path).encode()
    rc = lib.snx_libsvm_scan(bpath, ctypes.byref(n), ctypes.byref(nnz), ctypes.byref(mx))
    if rc != 0:
        msg = lib.snx_last_error().decode(errors="replace")
        if rc == 2:
            m = re.match(r"line (\d+): (.*)", msg, re.S)
            raise ParseError(m.group(2), int(m.group(1))) if m else ParseError(msg)
        raise OSError(msg)
    labels = np.empty(n.value, dtype=np.float64)
    indptr = np.empty(n.value + 1, dtype=np.int64)
    indices = np.empty(nnz.value, dtype=np.int32)
    data = np.empty(nnz.value, dtype=np.float64)
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _lib.call("snx_libsvm_fetch", bpath, ptr(labels), ptr(indptr), ptr(indices), ptr(data))
    return labels, indptr, indices, data, int(mx.value)


def load_libsvm(path, n_classes, n_features=None, storage="auto", dtype="f64"):
    """LIBSVM/svmlight file -> device dataset (dataset.py:242-293)."""
    csr, labels = parse_libsvm(path, n_classes, n_features)
    return _to_device(csr, labels, n_classes, storage, dtype)


def parse_csv(path, n_classes):
    """Host part of load_csv (dataset.py:298-311): (features n x p, 0-based
    labels); the empty table gives a 0 x 0 matrix; ParseError on malformed
    text, DataError on more distinct labels than classes."""
    import warnings

    with warnings.catch_warnings():  # numpy warns on an empty file; the reference too
        warnings.simplefilter("ignore", UserWarning)
        try:
            table = np.loadtxt(path, delimiter=",", dtype=np.float64, ndmin=2)
        except ValueError as exc:
            raise ParseError(str(exc)) from None
    if table.size == 0:
        return np.zeros((0, 0)), np.zeros(0, dtype=np.int64)
    return table[:, :-1], remap_labels(table[:, -1], n_classes)


def load_csv(path, n_classes, storage="dense", dtype="f64"):
    """Dense CSV, last column = label (dataset.py:296-311) -> device dataset."""
    import scipy.sparse as sp

    features, labels = parse_csv(path, n_classes)
    if features.size == 0 and len(labels) == 0:
        return DeviceDataset.from_numpy(features, labels, n_classes, dtype=dtype)
    return _to_device(sp.csr_array(features), labels, n_classes, storage, dtype)


__all__ = ["load_libsvm", "load_csv", "read_libsvm", "parse_libsvm", "parse_csv",
           "picks_dense", "remap_labels"]
