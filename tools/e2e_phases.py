import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_1802_09113_b200 as snx
from paper_1802_09113_b200 import sampling, device
N, P, C = 50000, 3072, 10
A, y = oracle.synthetic_problem(N, P, C, seed=0)
ds = snx.DeviceDataset.from_numpy(A, y, C)
prob = snx.SoftmaxProblem(ds, 1e-3)
x = 0.01 * np.random.default_rng(7).standard_normal((C - 1) * P)
g = np.random.default_rng(8).standard_normal((C - 1) * P)
cfg = snx.CgConfig(1e-4, 10)
for k in range(5):
    snx.cg_solve(snx.SubsampledOracle(prob, snx.SampleConfig(1.0, 0.05), k).hessian_operator(x), g, cfg)
torch.cuda.synchronize()
T = {}
def tick(name, t0):
    T[name] = T.get(name, 0) + time.perf_counter() - t0
    return time.perf_counter()
R = 50
for k in range(R):
    t = time.perf_counter()
    s_h = sampling.draw_index_set(0, 200 + k, 1, N, 2500, False); t = tick("draw_index_set", t)
    v = ds.take(s_h); t = tick("take+upload", t)
    w, _ = device.vec_in(x, ds.dim); t = tick("vec_in x", t)
    op = snx.softmax.HessianOperator(v, w, 1e-3, scale=N / 2500); t = tick("HessianOperator", t)
    gd, _ = device.vec_in(g, ds.dim); t = tick("vec_in g", t)
    ws = snx.cg.cg_graph_for(op, 10, 1e-4).run(gd); t = tick("graph run", t)
    st, sol = device.download(ws.slot(10), ws.pb); t = tick("download(sync)", t)
print({k: round(v / R * 1e6, 1) for k, v in T.items()})
