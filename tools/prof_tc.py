"""Profiling driver: the f32 tensor-core Hessian product at CIFAR shape (C = 10,
tc_gemm1/2) and on a config #5 shard (C = 100, tcw_gemm1/2), a few applies each
(for ncu: tensor-pipe utilisation of the tcgen05 GEMMs)."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_09113_b200 as snx  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "both"
if which in ("both", "c10"):
    n, p, C = 50000, 3072, 10
    gen = np.random.default_rng(0)
    A = gen.standard_normal((n, p))
    A /= np.sqrt((A ** 2).sum(axis=0))
    y = gen.integers(0, C, size=n)
    prob = snx.SoftmaxProblem(snx.DeviceDataset.from_numpy(A, y, C, dtype="f32"), 1e-3)
    x = torch.from_numpy(0.01 * gen.standard_normal((C - 1) * p)).cuda()
    op = snx.SubsampledOracle(prob, snx.SampleConfig(1.0, 0.05), 0).hessian_operator(x)
    out = torch.empty_like(x)
    for _ in range(6):
        op.apply_into(x, out)
    torch.cuda.synchronize()
    del prob, op
if which in ("both", "c100"):
    n, p, C = 1_000_000, 3072, 100
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.randn((n, p), generator=g, device="cuda", dtype=torch.float32).mul_(1 / math.sqrt(n))
    lab = torch.randint(0, C, (n,), generator=g, device="cuda", dtype=torch.int32)
    ds = snx.DeviceDataset(X, lab, C, p, dtype="f32")
    x = 0.05 * torch.randn((C - 1) * p, generator=g, device="cuda", dtype=torch.float64)
    view = ds.take(snx.draw_samples(snx.SampleConfig(1.0, 0.05), n, 0)[1])
    op = snx.HessianOperator(view, x, 1e-3, scale=n / view.n_rows)
    out = torch.empty_like(x)
    for _ in range(6):
        op.apply_into(x, out)
    torch.cuda.synchronize()
print("done")
