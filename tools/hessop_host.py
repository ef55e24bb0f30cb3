import os, sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import oracle
import paper_1802_09113_b200 as snx
from paper_1802_09113_b200 import device, softmax, _lib
from paper_1802_09113_b200.device import ptr, stream_handle
N, P, C = 50000, 3072, 10
A, y = oracle.synthetic_problem(N, P, C, seed=0)
ds = snx.DeviceDataset.from_numpy(A, y, C)
x = 0.01 * np.random.default_rng(7).standard_normal((C - 1) * P)
idx = np.sort(np.random.default_rng(1).choice(N, 2500, replace=False))
v = ds.take(idx)
w, _ = device.vec_in(x, ds.dim)
for _ in range(5): softmax.HessianOperator(v, w, 1e-3, scale=20.0)
torch.cuda.synchronize()
T = {}
def tk(n, t0):
    t1 = time.perf_counter(); T[n] = T.get(n, 0) + t1 - t0; return t1
R = 100
for _ in range(R):
    t = time.perf_counter()
    view = softmax._view(v); t = tk("_view", t)
    ww, ft = device.vec_in(w, view.dim); t = tk("vec_in", t)
    wc = ww.clone(); t = tk("clone", t)
    hb = view.base.hess_buffers(view.n_rows, view.rows is not None); t = tk("hess_buffers", t)
    hb.rows[:view.n_rows].copy_(view.rows); t = tk("rows copy_", t)
    wsp = softmax._ws(view); t = tk("_ws", t)
    sh = stream_handle(); t = tk("stream_handle", t)
    base = view.base
    _lib.call("snx_hess_prepare", base.code, ptr(base.X), base.ld, ptr(hb.rows), view.n_rows,
              view.n_features, view.K, ptr(wc), None, base.ld, ptr(hb.h), *wsp, sh); t = tk("lib call", t)
    op = softmax.HessianOperator(v, w, 1e-3, scale=20.0); t = tk("whole HessianOperator", t)
torch.cuda.synchronize()
print({k: round(v_ / R * 1e6, 1) for k, v_ in T.items()})
