"""CPU-only checks: the C ABI library loads and exports every declared symbol;
host-side logic (sample draws, configs, line search, variants) matches the
reference's contract.  No kernel is launched here (no GPU in this container)."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_1802_09113_b200 as snx
from paper_1802_09113_b200 import _build, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    _build.build()  # no-op when up to date (nvcc cross-compiles without a GPU)
    return _lib.load()


def header_functions():
    text = open(os.path.join(ROOT, "include", "snx.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(snx_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol(lib):
    names = header_functions()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} not bound in _lib.SIGNATURES"
    assert set(_lib.SIGNATURES) == set(names)


def test_library_is_sm100a(lib):
    out = os.popen(f"cuobjdump --list-elf {_build.LIBPATH} 2>&1").read()
    assert "sm_100a" in out, out


def test_abi_version_and_workspace(lib):
    assert lib.snx_abi_version() == 1
    a = _lib.workspace_bytes(_lib.F64, 50000, 3072, 9)
    b = _lib.workspace_bytes(_lib.F32, 50000, 3072, 9)
    assert a > 50000 * 9 * 8 and b > 50000 * 9 * 4
    assert _lib.workspace_bytes(_lib.F64, 0, 54, 6) > 0


def test_abi_errors_without_device(lib):
    # argument validation fails before any launch
    rc = lib.snx_objective(7, None, 4, 0, 4, 3, None, None, None, 0.0, None, None, None, 0,
                           None)
    assert rc != 0
    rc = lib.snx_hess_apply(0, None, 4, 10, 4, 40, ctypes.c_void_p(8), ctypes.c_void_p(8), 1.0,
                            0.0, ctypes.c_void_p(8), None, None, None, 0, None)
    assert rc != 0 and b"K = C-1" in lib.snx_last_error()


def test_device_required_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        snx.DeviceDataset.from_numpy(np.zeros((3, 4)), [0, 1, 0], 2)


def test_draw_samples_bit_exact(sampling_golden):
    g = sampling_golden
    i = 0
    while f"s{i}_params" in g:
        fg, fh, rep, seed, n, it = g[f"s{i}_params"]
        cfg = snx.SampleConfig(fg, fh, bool(rep), int(seed))
        s_g, s_h = snx.draw_samples(cfg, int(n), int(it))
        assert np.array_equal(s_h, g[f"s{i}_s_h"])
        if not bool(g[f"s{i}_s_g_full"]):
            assert np.array_equal(s_g, g[f"s{i}_s_g"])
        else:
            assert np.array_equal(s_g, np.arange(int(n)))
        i += 1
    assert snx.sample_size(0.05, 581012) == 29051
    with pytest.raises(snx.DataError):
        snx.draw_samples(snx.SampleConfig(), 0, 0)


def test_configs_validate():
    with pytest.raises(snx.DataError):
        snx.SampleConfig(gradient_fraction=0.0)
    with pytest.raises(snx.DataError):
        snx.SampleConfig(hessian_fraction=1.5)
    with pytest.raises(snx.DataError):
        snx.CgConfig(theta=1.0)
    with pytest.raises(snx.DataError):
        snx.CgConfig(max_iters=0)
    with pytest.raises(snx.DataError):
        snx.LineSearchConfig(beta=0.0)
    with pytest.raises(snx.DataError):
        snx.LineSearchConfig(rho=1.0)
    with pytest.raises(snx.DataError):
        snx.NewtonConfig(epsilon=0.0)
    with pytest.raises(snx.DataError):
        snx.TrustRegionConfig(eta=0.3)


def test_make_variant():
    for name, fr in snx.VARIANT_FRACTIONS.items():
        cfg = snx.make_variant(name, snx.NewtonConfig(epsilon=1e-5))
        assert (cfg.samples.gradient_fraction, cfg.samples.hessian_fraction) == fr
        assert cfg.epsilon == 1e-5
    with pytest.raises(ValueError):
        snx.make_variant("sorta-sampled")


def test_line_search_semantics(solver_golden):
    g = solver_golden
    for i in range(3):
        vals = list(g[f"ls{i}_vals"])
        f0, slope, alpha, evals = g[f"ls{i}_result"]
        seq = iter(vals)
        assert snx.line_search(lambda a: next(seq), f0, slope) == (alpha, int(evals))
    with pytest.raises(snx.LineSearchError):
        snx.line_search(lambda a: 0.0, 1.0, 0.0)
    with pytest.raises(snx.LineSearchError):
        snx.line_search(lambda a: 0.0, math.inf, -1.0)
    calls = []
    with pytest.raises(snx.LineSearchError):
        snx.line_search(lambda a: calls.append(a) or 5.0, 1.0, -1.0,
                        snx.LineSearchConfig(max_iters=4))
    assert len(calls) == 5 and calls[-1] == 0.0625


def test_error_hierarchy():
    for cls in (snx.ParseError, snx.DataError, snx.DimensionError, snx.CurvatureError,
                snx.LineSearchError):
        assert issubclass(cls, snx.SubnewtonError)
    assert "line 3" in str(snx.ParseError("bad", 3))
