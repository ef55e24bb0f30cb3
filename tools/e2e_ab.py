import os, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import bench
import paper_1802_09113_b200 as snx
from paper_1802_09113_b200 import sampling
A, y = bench.make_problem()
prob = snx.SoftmaxProblem(snx.DeviceDataset.from_numpy(A, y, 10), 1e-3)
x = 0.01 * np.random.default_rng(7).standard_normal(9 * 3072)
g = np.random.default_rng(8).standard_normal(9 * 3072)
cfg = snx.CgConfig(1e-4, 10)
def run(k0):
    t = time.perf_counter(); n = 0
    for k in range(k0, k0 + 60):
        n += snx.cg_solve(snx.SubsampledOracle(prob, snx.SampleConfig(1.0, 0.05), k).hessian_operator(x), g, cfg).iterations
    return n / (time.perf_counter() - t)
run(0)
print("lookahead on ", run(100))
orig = sampling._draw_ahead
sampling._draw_ahead = lambda key: None
run(300)
print("lookahead off", run(400))
sampling._draw_ahead = orig
print("lookahead on ", run(600))
