"""ctypes binding of libsnx (include/snx.h).

The product path has no CPU fallback: if the shared object is missing or a
CUDA device is absent, every entry point raises.  Device buffers are owned
by torch tensors; only raw pointers cross the ABI.
"""

import ctypes
import os

from ._build import LIBPATH

F64 = 0
F32 = 1
DOT_BLOCKS = 256
CG_SLOT = 8
POWER_STATE = 4 + 2 * DOT_BLOCKS
ABI_VERSION = 1

_c_int, _c_i32, _c_i64 = ctypes.c_int, ctypes.c_int32, ctypes.c_int64
_c_dbl, _c_size, _c_p = ctypes.c_double, ctypes.c_size_t, ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/snx.h one to one
SIGNATURES = {
    "snx_abi_version": (_c_int, []),
    "snx_last_error": (ctypes.c_char_p, []),
    "snx_workspace_bytes": (_c_size, [_c_int, _c_i64, _c_i32, _c_i32]),
    "snx_gather_rows": (_c_int, [_c_int, _c_p, _c_i64, _c_p, _c_p, _c_i64, _c_p, _c_i64, _c_p,
                                 _c_p]),
    "snx_objective": (_c_int, [_c_int, _c_p, _c_i64, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p,
                               _c_dbl, _c_p, _c_p, _c_p, _c_size, _c_p]),
    "snx_objective_grad": (_c_int, [_c_int, _c_p, _c_i64, _c_i64, _c_i32, _c_i32, _c_p, _c_p,
                                    _c_dbl, _c_dbl, _c_p, _c_p, _c_p, _c_size, _c_p]),
    "snx_objective_grad_acc": (_c_int, [_c_int, _c_p, _c_i64, _c_i64, _c_i32, _c_i32, _c_p, _c_p,
                                        _c_dbl, _c_dbl, _c_p, _c_p, _c_p, _c_p, _c_size, _c_p]),
    "snx_class_probabilities": (_c_int, [_c_int, _c_p, _c_i64, _c_i64, _c_i32, _c_i32, _c_p, _c_p,
                                         _c_p, _c_p, _c_p, _c_p, _c_size, _c_p]),
    "snx_csr_class_probabilities": (_c_int, [_c_p, _c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p,
                                             _c_p, _c_p, _c_p, _c_p, _c_size, _c_p]),
    "snx_hess_prepare": (_c_int, [_c_int, _c_p, _c_i64, _c_p, _c_i64, _c_i32, _c_i32, _c_p,
                                  _c_p, _c_i64, _c_p, _c_p, _c_size, _c_p]),
    "snx_hess_apply": (_c_int, [_c_int, _c_p, _c_i64, _c_i64, _c_i32, _c_i32, _c_p, _c_p,
                                _c_dbl, _c_dbl, _c_p, _c_p, _c_p, _c_p, _c_size, _c_p]),
    "snx_rowpass_fused": (_c_int, [_c_int, _c_i32, _c_i32]),
    "snx_hess_apply_rows": (_c_int, [_c_int, _c_p, _c_i64, _c_p, _c_i64, _c_i32, _c_i32, _c_p,
                                     _c_p, _c_dbl, _c_dbl, _c_p, _c_p, _c_p, _c_p, _c_size,
                                     _c_p]),
    "snx_hess_apply_cg_rows": (_c_int, [_c_int, _c_p, _c_i64, _c_p, _c_i64, _c_i32, _c_i32, _c_p,
                                        _c_dbl, _c_dbl, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p,
                                        _c_p, _c_p, _c_p, _c_size, _c_p]),
    "snx_tc_ld": (_c_i64, [_c_i32]),
    "snx_wide_scratch_doubles": (_c_i64, [_c_i64, _c_i32, _c_i32, _c_i64]),
    "snx_wide_objective": (_c_int, [_c_p, _c_i64, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p,
                                    _c_dbl, _c_p, _c_p, _c_p, _c_i64, _c_p]),
    "snx_wide_objective_grad": (_c_int, [_c_p, _c_i64, _c_i64, _c_i32, _c_i32, _c_p, _c_p,
                                         _c_dbl, _c_dbl, _c_p, _c_p, _c_p, _c_i64, _c_p]),
    "snx_wide_hess_prepare": (_c_int, [_c_p, _c_i64, _c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p,
                                       _c_i64, _c_p, _c_p, _c_i64, _c_p]),
    "snx_wide_hess_apply": (_c_int, [_c_p, _c_i64, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_dbl,
                                     _c_dbl, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_p]),
    "snx_wide_class_probabilities": (_c_int, [_c_p, _c_i64, _c_i64, _c_i32, _c_i32, _c_p, _c_p,
                                              _c_p, _c_p, _c_p, _c_p, _c_i64, _c_p]),
    "snx_wide_f32_scratch_doubles": (_c_i64, [_c_i64, _c_i32, _c_i32, _c_i64]),
    "snx_wide_class_probabilities_f32": (_c_int, [_c_p, _c_i64, _c_i64, _c_i32, _c_i32, _c_p,
                                                  _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_p]),
    "snx_hess_prepare_tc": (_c_int, [_c_p, _c_i64, _c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p,
                                     _c_i64, _c_p, _c_p, _c_p, _c_i64, _c_p, _c_size, _c_p]),
    "snx_hess_apply_tc": (_c_int, [_c_p, _c_p, _c_i64, _c_i64, _c_i32, _c_i32, _c_p, _c_p,
                                   _c_dbl, _c_dbl, _c_p, _c_p, _c_p, _c_p, _c_size, _c_p]),
    "snx_tc_split": (_c_int, [_c_p, _c_i64, _c_i64, _c_i32, _c_p, _c_p, _c_i64, _c_p]),
    "snx_objective_tc": (_c_int, [_c_p, _c_p, _c_i64, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p,
                                  _c_dbl, _c_p, _c_p, _c_p, _c_size, _c_p]),
    "snx_objective_grad_tc": (_c_int, [_c_p, _c_p, _c_i64, _c_i64, _c_i32, _c_i32, _c_p, _c_p,
                                       _c_dbl, _c_dbl, _c_p, _c_p, _c_p, _c_size, _c_p]),
    "snx_dot": (_c_int, [_c_p, _c_p, _c_i64, _c_p, _c_p]),
    "snx_dot_partials": (_c_int, [_c_p, _c_p, _c_i64, _c_p, _c_p]),
    "snx_axpy": (_c_int, [_c_p, _c_p, _c_dbl, _c_i64, _c_p, _c_p]),
    "snx_axpby": (_c_int, [_c_dbl, _c_p, _c_dbl, _c_p, _c_i64, _c_p, _c_p]),
    "snx_finish_hv": (_c_int, [_c_p, _c_dbl, _c_i64, _c_p, _c_p, _c_p, _c_p]),
    "snx_cg_init": (_c_int, [_c_p, _c_i64, _c_dbl, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p]),
    "snx_cg_update": (_c_int, [_c_i32, _c_i32, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p,
                               _c_p]),
    "snx_cg_done_flag": (_c_p, [_c_p, _c_i32]),
    "snx_power_step": (_c_int, [_c_p, _c_p, _c_i64, _c_p, _c_p]),
    "snx_colnorm_workspace_bytes": (_c_size, [_c_i32]),
    "snx_column_norms": (_c_int, [_c_int, _c_p, _c_i64, _c_i64, _c_i32, _c_p, _c_p, _c_p, _c_size,
                                  _c_p]),
    "snx_scale_columns": (_c_int, [_c_int, _c_p, _c_i64, _c_i64, _c_i32, _c_i64, _c_p, _c_p,
                                   _c_i64, _c_p]),
    "snx_csr_workspace_bytes": (_c_size, [_c_i64, _c_i32, _c_i32]),
    "snx_csr_objective": (_c_int, [_c_p, _c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p,
                                   _c_dbl, _c_p, _c_p, _c_p, _c_size, _c_p]),
    "snx_csr_objective_grad": (_c_int, [_c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_i32,
                                        _c_i32, _c_p, _c_p, _c_dbl, _c_dbl, _c_p, _c_p, _c_p,
                                        _c_size, _c_p]),
    "snx_csr_column_norms": (_c_int, [_c_p, _c_p, _c_i32, _c_p, _c_p, _c_p]),
    "snx_csr_scale_columns": (_c_int, [_c_p, _c_p, _c_p, _c_p, _c_i64, _c_i32, _c_p, _c_p, _c_p,
                                       _c_p, _c_p]),
    "snx_csr_gather": (_c_int, [_c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_i32, _c_p, _c_i64,
                                _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_size, _c_p]),
    "snx_csr_hess_prepare": (_c_int, [_c_p, _c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p,
                                      _c_size, _c_p]),
    "snx_csr_hess_apply": (_c_int, [_c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_i32, _c_i32,
                                    _c_p, _c_p, _c_dbl, _c_dbl, _c_p, _c_p, _c_p, _c_p, _c_size,
                                    _c_p]),
    "snx_libsvm_scan": (_c_int, [ctypes.c_char_p, _c_p, _c_p, _c_p]),
    "snx_libsvm_fetch": (_c_int, [ctypes.c_char_p, _c_p, _c_p, _c_p, _c_p]),
    "snx_tr_init": (_c_int, [_c_p, _c_i64, _c_dbl, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_p]),
    "snx_tr_update": (_c_int, [_c_i32, _c_i32, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p,
                               _c_p, _c_p]),
    "snx_pack_rows": (_c_int, [_c_int, _c_p, _c_i64, _c_i32, _c_p, _c_i64, _c_p]),
}

_lib = None


class SnxError(RuntimeError):
    """A libsnx call returned non-zero (message from snx_last_error)."""


def load():
    """Load libsnx.so (built by __graft_entry__.build()); fail loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("SNX_LIB", LIBPATH)  # debug builds (tools/timeline.py)
    if not os.path.exists(path):
        raise ImportError(
            f"libsnx CUDA extension not built ({LIBPATH} missing): run "
            "`python -c 'import __graft_entry__ as g; g.build()'` -- there is no CPU fallback")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.snx_abi_version() != ABI_VERSION:
        raise ImportError(f"libsnx ABI {lib.snx_abi_version()} != expected {ABI_VERSION}")
    _lib = lib
    return lib


def call(name, *args):
    """Invoke an int-returning entry point; raise SnxError on failure."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        raise SnxError(lib.snx_last_error().decode(errors="replace"))
    return rc


def workspace_bytes(dtype, nrows, P, K):
    return int(load().snx_workspace_bytes(dtype, nrows, P, K))


def done_flag(state_ptr, t):
    return load().snx_cg_done_flag(state_ptr, t)
