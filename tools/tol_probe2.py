import math, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1802_09113_b200 as snx
from paper_1802_09113_b200 import softmax
from paper_1802_09113_b200.device import dot
from tol_probe import planted
import oracle
for lbl in ["planted", "uniform"]:
    if lbl == "planted":
        A, y = planted(50000, 3072, 10, scale=3.0)
    else:
        A, y = oracle.synthetic_problem(50000, 3072, 10, seed=0)
    ds = snx.DeviceDataset.from_numpy(A, y, 10)
    prob = snx.SoftmaxProblem(ds, 1e-3)
    x0 = torch.zeros(9 * 3072, dtype=torch.float64, device="cuda")
    g0 = math.sqrt(float(dot(*(2 * [softmax.gradient_parts(ds, x0, 1.0, 1e-3)[0]]))))
    for rel in [1e-2, 1e-3, 1e-4, 1e-5]:
        cfg = snx.make_variant("subsampled-100", snx.NewtonConfig(epsilon=rel * g0, max_outer_iters=300))
        torch.cuda.synchronize(); t = time.perf_counter()
        tr = snx.newton_solve(prob, cfg, x0=x0.clone())
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(lbl, rel, tr.reason, tr.iterations, round(dt, 4), tr.final_objective)
