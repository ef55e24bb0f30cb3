"""Newton iteration time with frequent Armijo backtracking (alpha0 = 64 on a
planted CIFAR-shape problem: every iteration backtracks 64 -> 32 -> 16), per
speculation policy (a discarded speculative iteration must not sit
in front of every Armijo trial).

    SNX_SPECULATE=adaptive|always|never python tools/backtrack_timing.py
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_09113_b200 as snx  # noqa: E402

n, p, C = 50000, 3072, 10
gen = np.random.default_rng(5)
A = gen.standard_normal((n, p))
A /= np.sqrt((A ** 2).sum(axis=0))
y = (A @ (10.0 * gen.standard_normal((p, C)))).argmax(axis=1).astype(np.int64)
prob = snx.SoftmaxProblem(snx.DeviceDataset.from_numpy(A, y, C), 1e-4)
for a0, variant in ((64.0, "subsampled-20"), (1.0, "subsampled-100")):
    cfg = snx.make_variant(variant, snx.NewtonConfig(max_outer_iters=12,
                                                     ls=snx.LineSearchConfig(alpha0=a0)))
    snx.newton_solve(prob, cfg)  # warm-up (graph capture)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr = snx.newton_solve(prob, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{os.environ.get('SNX_SPECULATE', 'adaptive'):8s} {variant} alpha0={a0:g}: "
          f"{1e3 * dt / tr.iterations:.3f} ms/iter, steps {[r.step_size for r in tr.records[1:]]}")
