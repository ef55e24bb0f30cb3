"""Per-kernel times of the CSR passes at the Newsgroups20 shape (ncu target)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_1802_09113_b200 import softmax
from paper_1802_09113_b200.sparse import CsrDataset
A, y = bench.sparse_problem()
ds = CsrDataset.from_scipy(A, y, 20)
x = torch.from_numpy(0.01 * np.random.default_rng(7).standard_normal(19 * A.shape[1])).cuda()
for _ in range(3):
    g, _ = softmax.gradient_parts(ds, x, 1.0, 1e-3)
torch.cuda.synchronize()
