import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def softmax_golden():
    return load_golden("softmax_golden.npz")


@pytest.fixture(scope="session")
def sampling_golden():
    return load_golden("sampling_golden.npz")


@pytest.fixture(scope="session")
def solver_golden():
    return load_golden("solver_golden.npz")


def softmax_cases(g):
    i = 0
    while f"c{i}_shape" in g:
        yield i, {k[len(f"c{i}_"):]: v for k, v in g.items() if k.startswith(f"c{i}_")}
        i += 1


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    num = np.linalg.norm(a - b)
    return num if den == 0 else num / den


@pytest.fixture(scope="session")
def cuda_ok():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True


@pytest.fixture(scope="session")
def data_golden():
    return load_golden("data_golden.npz")


@pytest.fixture(scope="session")
def sparse_golden():
    return load_golden("sparse_golden.npz")


def sparse_cases(g):
    import scipy.sparse as sp

    i = 0
    while f"s{i}_shape" in g:
        n, p, C = (int(t) for t in g[f"s{i}_shape"])
        A = sp.csr_array((g[f"s{i}_data"], g[f"s{i}_indices"], g[f"s{i}_indptr"]), shape=(n, p))
        yield i, A, C, {k[len(f"s{i}_"):]: v for k, v in g.items() if k.startswith(f"s{i}_")}
        i += 1


@pytest.fixture(scope="session")
def libsvm_golden():
    return load_golden("libsvm_golden.npz")


def libsvm_cases(g):
    names = sorted({k[:-len("_args")] for k in g if k.endswith("_args")})
    for name in names:
        C, nf = (int(t) for t in g[name + "_args"])
        yield name, os.path.join(GOLDEN, "libsvm", name + ".svm"), C, (None if nf < 0 else nf), \
            str(g[name + "_storage"]), {k[len(name) + 1:]: v for k, v in g.items()
                                         if k.startswith(name + "_")}
