"""ncu target for the 8(f) kernels: CSR Hessian product (Newsgroups20 shape),
one power-iteration step at CIFAR shape, one Steihaug-CG solve."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import oracle
import paper_1802_09113_b200 as snx
from paper_1802_09113_b200 import softmax
from paper_1802_09113_b200.sparse import CsrDataset
A, y = bench.sparse_problem()
ds = CsrDataset.from_scipy(A, y, 20)
x = torch.from_numpy(0.01 * np.random.default_rng(7).standard_normal(19 * A.shape[1])).cuda()
orc = snx.SubsampledOracle(snx.SoftmaxProblem(ds, 1e-3), snx.SampleConfig(1.0, 0.05), 0)
op = orc.hessian_operator(x)
out = torch.empty_like(x)
for _ in range(3):
    op.apply_into(x, out)
A2, y2 = oracle.synthetic_problem(50000, 3072, 10, seed=0)
d2 = snx.DeviceDataset.from_numpy(A2, y2, 10)
snx.estimate_lipschitz(snx.SoftmaxProblem(d2, 0.0), iters=2)
x2 = torch.from_numpy(0.01 * np.random.default_rng(7).standard_normal(9 * 3072)).cuda()
o2 = snx.SubsampledOracle(snx.SoftmaxProblem(d2, 1e-3), snx.SampleConfig(1.0, 0.1), 0)
g2 = o2.gradient_device(x2)[0]
snx.steihaug_cg(o2.hessian_operator(x2), g2, 1.0, 1e-4, 10)
torch.cuda.synchronize()
