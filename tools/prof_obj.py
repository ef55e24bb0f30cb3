"""Profiling driver: CIFAR-shape full objective + gradient passes (for ncu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1802_09113_b200 as snx  # noqa: E402
from paper_1802_09113_b200 import softmax  # noqa: E402

dtype = sys.argv[1] if len(sys.argv) > 1 else "f64"
A, y = oracle.synthetic_problem(50000, 3072, 10, seed=0)
ds = snx.DeviceDataset.from_numpy(A, y, 10, dtype=dtype)
x = torch.from_numpy(0.01 * np.random.default_rng(7).standard_normal(9 * 3072)).cuda()
for _ in range(3):
    softmax.objective_parts(ds, x, want_correct=True)
for _ in range(2):
    softmax.gradient_parts(ds, x, 1.0, 1e-3)
torch.cuda.synchronize()
print("ok")
