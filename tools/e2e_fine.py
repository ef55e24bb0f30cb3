"""Host-side anatomy of one e2e bench step through the public API (pinned host
tensors in, the solution back into pinned host memory): wall time between the
API boundaries, no extra synchronisation.

    python tools/e2e_fine.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1802_09113_b200 as snx  # noqa: E402

N, P, C = 50000, 3072, 10
A, y = oracle.synthetic_problem(N, P, C, seed=0)
ds = snx.DeviceDataset.from_numpy(A, y, C)
prob = snx.SoftmaxProblem(ds, 1e-3)
x = torch.from_numpy(0.01 * np.random.default_rng(7).standard_normal((C - 1) * P)).pin_memory()
g = torch.from_numpy(np.random.default_rng(8).standard_normal((C - 1) * P)).pin_memory()
out = torch.empty_like(g).pin_memory()
cfg = snx.CgConfig(1e-4, 10)
sc = snx.SampleConfig(1.0, 0.05)


def step(k, T=None):
    t = time.perf_counter()
    orc = snx.SubsampledOracle(prob, sc, k)
    t1 = time.perf_counter()
    op = orc.hessian_operator(x)
    t2 = time.perf_counter()
    rep = snx.cg_solve(op, g, cfg)
    t3 = time.perf_counter()
    out.copy_(rep.solution, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    t4 = time.perf_counter()
    if T is not None:
        for name, v in (("oracle", t1 - t), ("hessian_operator", t2 - t1), ("cg_solve", t3 - t2),
                        ("result copy + sync", t4 - t3)):
            T[name] = T.get(name, 0) + v


for k in range(5):
    step(k)
torch.cuda.synchronize()
T = {}
R = 50
for k in range(R):
    step(100 + k, T)
print({k: round(v / R * 1e6, 1) for k, v in T.items()}, "total", round(sum(T.values()) / R * 1e6, 1))
import cProfile  # noqa: E402
import pstats  # noqa: E402

pr = cProfile.Profile()
pr.enable()
for k in range(R):
    step(300 + k)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
