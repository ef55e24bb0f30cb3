"""Timeline of the last CG iteration of a captured CG solve (debug build):
first entry / last exit of every kernel and the gaps between them.

    python -c "from paper_1802_09113_b200 import _build; _build.build_timeline('tools/libsnx_tl.so')"
    SNX_LIB=tools/libsnx_tl.so python tools/timeline_cg.py [f64]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1802_09113_b200 as snx  # noqa: E402
from paper_1802_09113_b200 import _lib, cg as cgmod  # noqa: E402

dtype = sys.argv[1] if len(sys.argv) > 1 else "f64"
A, y = oracle.synthetic_problem(50000, 3072, 10, seed=0)
ds = snx.DeviceDataset.from_numpy(A, y, 10, dtype=dtype)
x = torch.from_numpy(0.01 * np.random.default_rng(7).standard_normal(9 * 3072)).cuda()
orc = snx.SubsampledOracle(snx.SoftmaxProblem(ds, 1e-3), snx.SampleConfig(1.0, 0.05), 0)
g, _ = orc.gradient_device(x)
op = orc.hessian_operator(x)
for _ in range(3):
    ws = cgmod.cg_graph_for(op, 10, 1e-4).run(g)
torch.cuda.synchronize()
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
ws = cgmod.cg_graph_for(op, 10, 1e-4).run(g)
e1.record(st)
torch.cuda.synchronize()
print(f"cg graph: {e0.elapsed_time(e1) * 1e3:.1f} us, iterations {int(ws.slot(10)[3])}")
lib = _lib.load()
rows = []
if dtype == "f32":
    b = (ctypes.c_ulonglong * (2 * 160 * 8))()
    assert lib.snx_debug_tc_timeline(b) == 0
    t = np.frombuffer(b, dtype=np.uint64).reshape(2, 160, 8).astype(np.int64)
    rows += [("tc_gemm1", t[0, :, 0], t[0, :, 3]), ("tc_gemm2", t[1, :, 0], t[1, :, 3])]
else:
    b = (ctypes.c_ulonglong * (3 * 160 * 8))()
    assert lib.snx_debug_timeline(b) == 0
    t = np.frombuffer(b, dtype=np.uint64).reshape(3, 160, 8).astype(np.int64)
    rows += [("gemm1", t[0, :, 0], t[0, :, 3]), ("gemm2", t[1, :, 0], t[1, :, 3])]
b = (ctypes.c_ulonglong * (3 * 160 * 8))()
assert lib.snx_debug_timeline(b) == 0
t = np.frombuffer(b, dtype=np.uint64).reshape(3, 160, 8).astype(np.int64)
rows.append(("finalize", t[2, :, 0], t[2, :, 3]))
vb = (ctypes.c_ulonglong * (2 * 256 * 2))()
assert lib.snx_debug_vec_timeline(vb) == 0
v = np.frombuffer(vb, dtype=np.uint64).reshape(2, 256, 2).astype(np.int64)
rows += [("cg_step1", v[0, :, 0], v[0, :, 1]), ("cg_step2", v[1, :, 0], v[1, :, 1])]
rows = [r for r in rows if (r[1] > 0).any()]
base = min(r[1][r[1] > 0].min() for r in rows)
prev = None
for name, ent, ex in rows:
    ent, ex = ent[ent > 0], ex[ex > 0]
    e_min, e_med, x_med, x_max = ent.min(), np.median(ent), np.median(ex), ex.max()
    gap = (e_min - prev) / 1e3 if prev is not None else 0.0
    print(f"{name:9s} entry {(e_min - base) / 1e3:7.2f} (med {(e_med - base) / 1e3:7.2f})  "
          f"exit med {(x_med - base) / 1e3:7.2f} max {(x_max - base) / 1e3:7.2f}  "
          f"span {(x_max - e_min) / 1e3:6.2f} us  gap before {gap:5.2f}")
    prev = x_max
if dtype == "f64":
    names = ["entry", "1st data", "compute done", "exit", "seg written", "atomic", "epi0", "epi1"]
    for k, nm in enumerate(["gemm1", "gemm2"]):
        tt = t[k, :148].astype(np.float64)
        b0 = tt[:, 0].min()
        for ev in range(8):
            col = tt[:, ev]
            col = col[col > 0]
            if len(col):
                print(f"  {nm} {names[ev]:13s} n={len(col):3d} med {(np.median(col) - b0) / 1e3:7.2f}"
                      f" max {(col.max() - b0) / 1e3:7.2f}")
