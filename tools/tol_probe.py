"""Time-to-tolerance probe: planted-softmax labels at CIFAR shape."""
import math, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_09113_b200 as snx
from paper_1802_09113_b200 import softmax
from paper_1802_09113_b200.device import dot

def planted(n, p, C, seed=0, scale=3.0):
    g = np.random.default_rng(seed)
    A = g.standard_normal((n, p))
    A /= np.sqrt((A ** 2).sum(axis=0))
    W = g.standard_normal((p, C)) * scale
    Z = A @ W
    Z -= Z.max(axis=1, keepdims=True)
    P = np.exp(Z); P /= P.sum(axis=1, keepdims=True)
    u = g.random(n)[:, None]
    y = (P.cumsum(axis=1) < u).sum(axis=1).clip(0, C - 1)
    return A, y.astype(np.int64)

for scale in [float(s) for s in sys.argv[1:]] or [3.0]:
    A, y = planted(50000, 3072, 10, scale=scale)
    ds = snx.DeviceDataset.from_numpy(A, y, 10)
    prob = snx.SoftmaxProblem(ds, 1e-3)
    x0 = torch.zeros(9 * 3072, dtype=torch.float64, device="cuda")
    g0 = math.sqrt(float(dot(*(2 * [softmax.gradient_parts(ds, x0, 1.0, 1e-3)[0]]))))
    for variant in ["subsampled-100", "full"]:
        cfg = snx.make_variant(variant, snx.NewtonConfig(epsilon=1e-6 * g0, max_outer_iters=100))
        torch.cuda.synchronize(); t = time.perf_counter()
        tr = snx.newton_solve(prob, cfg, x0=x0.clone())
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(scale, variant, tr.reason, tr.iterations, round(dt, 4), tr.final_objective, [r.cg_iters for r in tr.records[1:]][:12])
