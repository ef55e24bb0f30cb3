"""Per-CTA timeline of the GEMM kernels of one Hessian product (debug build).

    python -c "from paper_1802_09113_b200 import _build; _build.build_timeline('tools/libsnx_tl.so')"
    SNX_LIB=tools/libsnx_tl.so python tools/timeline.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1802_09113_b200 as snx  # noqa: E402
from paper_1802_09113_b200 import _lib  # noqa: E402

A, y = oracle.synthetic_problem(50000, 3072, 10, seed=0)
ds = snx.DeviceDataset.from_numpy(A, y, 10, dtype=sys.argv[1] if len(sys.argv) > 1 else "f64")
x = torch.from_numpy(0.01 * np.random.default_rng(7).standard_normal(9 * 3072)).cuda()
orc = snx.SubsampledOracle(snx.SoftmaxProblem(ds, 1e-3), snx.SampleConfig(1.0, 0.05), 0)
g, _ = orc.gradient_device(x)
op = orc.hessian_operator(x)
out = torch.empty_like(g)
for _ in range(5):
    op.apply_into(g, out)
torch.cuda.synchronize()
op.apply_into(g, out)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (3 * 160 * 8))()
lib = _lib.load()
if ds.dtype == "f32":  # tensor-core kernels (snx_tc.cu)
    assert lib.snx_debug_tc_timeline(buf) == 0
    t = np.frombuffer(buf, dtype=np.uint64)[:2 * 160 * 8].reshape(2, 160, 8).astype(np.int64)
else:
    assert lib.snx_debug_timeline(buf) == 0
    t = np.frombuffer(buf, dtype=np.uint64).reshape(3, 160, 8).astype(np.int64)
for k, name in enumerate(["gemm1", "gemm2"]):
    tt = t[k, :148]
    tt = tt[tt[:, 0] > 0]
    base = tt[:, 0].min()
    rel = (tt - base) / 1e3
    print(f"{name}: entry   min/med/max {rel[:,0].min():7.2f} {np.median(rel[:,0]):7.2f} {rel[:,0].max():7.2f} us")
    print(f"{name}: 1st data min/med/max {rel[:,1].min():7.2f} {np.median(rel[:,1]):7.2f} {rel[:,1].max():7.2f}")
    print(f"{name}: compute done      {rel[:,2].min():7.2f} {np.median(rel[:,2]):7.2f} {rel[:,2].max():7.2f}")
    print(f"{name}: exit              {rel[:,3].min():7.2f} {np.median(rel[:,3]):7.2f} {rel[:,3].max():7.2f}")
g1x = t[0, :148, 3].max()
print("gemm2 entry - gemm1 last exit: %.2f us" % ((t[1, :148, 0].min() - g1x) / 1e3))
