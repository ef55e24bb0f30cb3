"""B200-native sub-sampled Newton-CG for L2-regularised softmax regression.

Drop-in for the hot path of the reference package `subnewton` (arXiv
1802.09113): same solver entry points, callables, configs, result objects and
exceptions; the arithmetic runs in hand-written sm_100a kernels (libsnx,
include/snx.h) called through ctypes.  torch only owns device memory.
"""

from .cg import CgConfig, CgReport, cg_solve
from .data import column_norms, normalize_columns, train_test_split
from .device import DeviceDataset, DeviceView, as_device
from .io import load_csv, load_libsvm
from .sparse import CsrDataset
from .errors import (CurvatureError, DataError, DimensionError, LineSearchError, ParseError,
                     SubnewtonError)
from .linesearch import LineSearchConfig, line_search
from .lipschitz import estimate_lipschitz
from .newton import VARIANT_FRACTIONS, NewtonConfig, make_variant, minimize, newton_solve
from .rng import stream_rng
from .sampling import SampleConfig, SubsampledOracle, draw_samples, sample_size
from .softmax import (BLOCK_ROWS, HessianOperator, RowStats, SoftmaxProblem, accuracy,
                      class_probabilities, data_gradient, data_objective, gradient, hess_vec,
                      matrix_as_weights, objective, predict, row_stats, weights_as_matrix,
                      zero_weights)
from .trace import RunRecord, SolveTrace, read_trace_csv, write_trace_csv
from .trust_region import TrustRegionConfig, steihaug_cg, trust_region_solve

__version__ = "0.1.0"

__all__ = [
    "CgConfig", "CgReport", "cg_solve", "DeviceDataset", "DeviceView", "as_device",
    "CurvatureError", "DataError", "DimensionError", "LineSearchError", "ParseError",
    "SubnewtonError", "LineSearchConfig", "line_search", "VARIANT_FRACTIONS", "NewtonConfig",
    "make_variant", "minimize", "newton_solve", "stream_rng", "SampleConfig",
    "SubsampledOracle", "draw_samples", "sample_size", "BLOCK_ROWS", "HessianOperator",
    "SoftmaxProblem", "accuracy", "data_gradient", "data_objective", "gradient", "hess_vec",
    "matrix_as_weights", "objective", "weights_as_matrix", "zero_weights", "RunRecord",
    "SolveTrace", "TrustRegionConfig", "steihaug_cg", "trust_region_solve",
    "estimate_lipschitz", "column_norms", "normalize_columns", "train_test_split",
    "read_trace_csv", "write_trace_csv", "load_libsvm", "load_csv", "RowStats", "row_stats",
    "class_probabilities", "predict", "CsrDataset",
]
