"""Where one iteration of the captured CG solve goes (debug build with both
timelines): the last product's CTAs (entry .. exit), cg_step1_rows (entry,
dependency met, exit) and cg_step2 (dependency met, exit), on one clock.

    python -c "from paper_1802_09113_b200 import _build; _build.build_timeline('tools/libsnx_cgtl.so', ['-DSNX_TIMELINE', '-DSNX_CL_TIMELINE'])"
    SNX_LIB=tools/libsnx_cgtl.so python tools/cg_iter_timeline.py [cifar|mnist]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_09113_b200 as snx  # noqa: E402
from paper_1802_09113_b200 import _lib, cg as cgmod  # noqa: E402

SHAPES = {"cifar": (50000, 3072, 10), "mnist": (60000, 784, 10)}
name = sys.argv[1] if len(sys.argv) > 1 else "cifar"
n, p, C = SHAPES[name]
gen = np.random.default_rng(0)
A = gen.standard_normal((n, p))
A /= np.sqrt((A ** 2).sum(axis=0))
y = gen.integers(0, C, size=n)
ds = snx.DeviceDataset.from_numpy(A, y, C)
x = torch.from_numpy(0.01 * np.random.default_rng(7).standard_normal((C - 1) * p)).cuda()
orc = snx.SubsampledOracle(snx.SoftmaxProblem(ds, 1e-3), snx.SampleConfig(1.0, 0.05), 0)
g, _ = orc.gradient_device(x)
op = orc.hessian_operator(x)
for _ in range(5):
    cgmod.cg_graph_for(op, 10, 1e-12).run(g)
torch.cuda.synchronize()
lib = _lib.load()
NB = 26
cl = (ctypes.c_ulonglong * (160 * NB * 10))()
lib.snx_debug_cl_timeline(cl)
cl = np.frombuffer(cl, dtype=np.uint64).reshape(160, NB, 10).astype(np.int64)
cr = (ctypes.c_ulonglong * (256 * 6))()
lib.snx_debug_cgr_timeline(cr)
cr = np.frombuffer(cr, dtype=np.uint64).reshape(256, 6).astype(np.int64)
vb = (ctypes.c_ulonglong * (2 * 256 * 2))()
lib.snx_debug_vec_timeline(vb)
v = np.frombuffer(vb, dtype=np.uint64).reshape(2, 256, 2).astype(np.int64)
used = [c for c in range(160) if cl[c, 0, 0] != 0]
ent = np.array([cl[c, 0, 0] for c in used])
pdl = np.array([cl[c, 0, 8] for c in used])
ext = np.array([cl[c, 0, 5] for c in used])
t0 = ent.min()
us = lambda a: (a - t0) / 1e3  # noqa: E731
print(f"{name}: product CTAs entry {us(ent.min()):6.2f}..{us(ent.max()):6.2f}  dependency met "
      f"{us(np.median(pdl)):6.2f}  exit med {us(np.median(ext)):6.2f} max {us(ext.max()):6.2f}")
print(f"cg_step1_rows   entry {us(cr[:, 0].min()):6.2f}..{us(cr[:, 0].max()):6.2f}  dependency met "
      f"{us(np.median(cr[:, 1])):6.2f}  exit med {us(np.median(cr[:, 2])):6.2f} max "
      f"{us(cr[:, 2].max()):6.2f}")
print("cg_step1_rows medians: loads+F-reduce " + f"{us(np.median(cr[:, 3])):6.2f}, alpha shared "
      f"{us(np.median(cr[:, 4])):6.2f}, element updates {us(np.median(cr[:, 5])):6.2f}")
print(f"cg_step2        dependency met {us(v[1, :, 0].min()):6.2f}..{us(np.median(v[1, :, 0])):6.2f}"
      f"  exit med {us(np.median(v[1, :, 1])):6.2f} max {us(v[1, :, 1].max()):6.2f}")
