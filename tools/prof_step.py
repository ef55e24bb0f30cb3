"""Host/device breakdown of one bench step (h-prep + graph CG)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1802_09113_b200 as snx  # noqa: E402
from paper_1802_09113_b200 import cg as cgmod, softmax  # noqa: E402

N, P, C = 50000, 3072, 10
A, y = oracle.synthetic_problem(N, P, C, seed=0)
ds = snx.DeviceDataset.from_numpy(A, y, C)
x = torch.from_numpy(0.01 * np.random.default_rng(7).standard_normal((C - 1) * P)).cuda()
g, _ = softmax.gradient_parts(ds, x, 1.0, 1e-3)
views = [ds.take(snx.draw_samples(snx.SampleConfig(1.0, 0.05), N, k)[1]) for k in range(30)]
st = torch.cuda.current_stream()


def timed(fn, reps=10):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    for k in range(reps):
        fn(k)
    e1.record(st)
    th = (time.perf_counter() - t0) / reps * 1e6
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3, th


ops = {}
for k in range(3):
    op = softmax.HessianOperator(views[k], x, 1e-3, scale=N / 2500)
    cgmod.cg_graph_for(op, 10, 1e-4).run(g)
print("prepare        gpu %.1f us  host %.1f us" % timed(lambda k: ops.__setitem__(0, softmax.HessianOperator(views[k], x, 1e-3, scale=N / 2500))))
op = ops[0]
print("cg graph run   gpu %.1f us  host %.1f us" % timed(lambda k: cgmod.cg_graph_for(op, 10, 1e-4).run(g)))
def full(k):
    o = softmax.HessianOperator(views[k], x, 1e-3, scale=N / 2500)
    cgmod.cg_graph_for(o, 10, 1e-4).run(g)
print("step           gpu %.1f us  host %.1f us" % timed(full))
import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
for k in range(10):
    full(k)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
