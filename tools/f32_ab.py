import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1802_09113_b200 as snx
from paper_1802_09113_b200 import device, cg as cgmod
n, p, C = 50000, 3072, 10
gen = np.random.default_rng(0)
A = gen.standard_normal((n, p)); A /= np.sqrt((A ** 2).sum(axis=0))
y = gen.integers(0, C, size=n)
for tc in (False, True):
    device.F32_TENSOR_CORES = tc
    ds = snx.DeviceDataset.from_numpy(A, y, C, dtype="f32")
    prob = snx.SoftmaxProblem(ds, 1e-3)
    x = torch.from_numpy(0.01 * np.random.default_rng(7).standard_normal((C - 1) * p)).cuda()
    orc = snx.SubsampledOracle(prob, snx.SampleConfig(1.0, 0.05), 0)
    g, _ = orc.gradient_device(x)
    op = orc.hessian_operator(x)
    out = torch.empty_like(g)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5): op.apply_into(g, out)
    torch.cuda.synchronize(); e0.record(st)
    for _ in range(100): op.apply_into(g, out)
    e1.record(st); torch.cuda.synchronize()
    hv = e0.elapsed_time(e1) / 100 * 1e3
    for _ in range(3): cgmod.cg_graph_for(op, 10, 1e-4).run(g)
    torch.cuda.synchronize(); e0.record(st)
    for _ in range(20): cgmod.cg_graph_for(op, 10, 1e-4).run(g)
    e1.record(st); torch.cuda.synchronize()
    cgt = e0.elapsed_time(e1) / 20 * 1e3
    for _ in range(3): snx.softmax.gradient_parts(ds, x, 1.0, 1e-3)
    torch.cuda.synchronize(); e0.record(st)
    for _ in range(10): snx.softmax.gradient_parts(ds, x, 1.0, 1e-3)
    e1.record(st); torch.cuda.synchronize()
    gr = e0.elapsed_time(e1) / 10 * 1e3
    print(f"f32 {'tcgen05' if tc else 'one-pass'}: hess_apply {hv:.1f} us | cg_solve(10) {cgt:.1f} us | full grad {gr:.1f} us", flush=True)
    del ds, prob, orc, op
    torch.cuda.empty_cache()
