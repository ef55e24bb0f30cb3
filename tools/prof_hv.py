"""Profiling driver: CIFAR-shape sampled Hessian operator, a few applies (for ncu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (synthetic data recipe)
import paper_1802_09113_b200 as snx  # noqa: E402

dtype = sys.argv[1] if len(sys.argv) > 1 else "f64"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
N, P, C = 50000, 3072, 10
A, y = oracle.synthetic_problem(N, P, C, seed=0)
ds = snx.DeviceDataset.from_numpy(A, y, C, dtype=dtype)
prob = snx.SoftmaxProblem(ds, 1e-3)
x = torch.from_numpy(0.01 * np.random.default_rng(7).standard_normal((C - 1) * P)).cuda()
orc = snx.SubsampledOracle(prob, snx.SampleConfig(1.0, 0.05), 0)
g, _ = orc.gradient_device(x)
op = orc.hessian_operator(x)
out = torch.empty_like(g)
for _ in range(reps):
    op.apply_into(g, out)
torch.cuda.synchronize()
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(20):
    op.apply_into(g, out)
e1.record(st)
torch.cuda.synchronize()
print(f"{dtype} hess_apply {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
e0.record(st)
for _ in range(5):
    snx.softmax.gradient_parts(ds, x, 1.0, 1e-3)
e1.record(st)
torch.cuda.synchronize()
print(f"{dtype} full gradient {e0.elapsed_time(e1) / 5 * 1e3:.1f} us")
e0.record(st)
for _ in range(5):
    snx.softmax.objective_parts(ds, x, g, 0.5, want_correct=True)
e1.record(st)
torch.cuda.synchronize()
print(f"{dtype} full objective+acc {e0.elapsed_time(e1) / 5 * 1e3:.1f} us")
from paper_1802_09113_b200 import cg as cgmod  # noqa: E402
for _ in range(3):
    ws = cgmod.cg_graph_for(op, 10, 1e-4).run(g)
torch.cuda.synchronize()
e0.record(st)
for _ in range(10):
    ws = cgmod.cg_graph_for(op, 10, 1e-4).run(g)
e1.record(st)
torch.cuda.synchronize()
print(f"{dtype} cg_solve (10 Hv) {e0.elapsed_time(e1) / 10 * 1e3:.1f} us, iters {ws.slot(10)[3].item()}")
e0.record(st)
for k in range(5):
    o2 = snx.SubsampledOracle(prob, snx.SampleConfig(1.0, 0.05), 100 + k)
    o2.hessian_operator(x)
e1.record(st)
torch.cuda.synchronize()
print(f"{dtype} oracle+hess_prepare {e0.elapsed_time(e1) / 5 * 1e3:.1f} us (incl. host draw)")
