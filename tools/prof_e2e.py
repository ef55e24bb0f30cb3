"""cProfile of the bench's e2e loop (public numpy API, host buffers)."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1802_09113_b200 as snx  # noqa: E402

N, P, C = 50000, 3072, 10
A, y = oracle.synthetic_problem(N, P, C, seed=0)
prob = snx.SoftmaxProblem(snx.DeviceDataset.from_numpy(A, y, C), 1e-3)
x = 0.01 * np.random.default_rng(7).standard_normal((C - 1) * P)
g = np.random.default_rng(8).standard_normal((C - 1) * P)
cfg = snx.CgConfig(1e-4, 10)


def step(k):
    orc = snx.SubsampledOracle(prob, snx.SampleConfig(1.0, 0.05), 500 + k)
    return snx.cg_solve(orc.hessian_operator(x), g, cfg)


for k in range(5):
    step(k)
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(20):
    step(k)
print("e2e step %.1f us" % ((time.perf_counter() - t0) / 20 * 1e6))
pr = cProfile.Profile()
pr.enable()
for k in range(20):
    step(k)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
