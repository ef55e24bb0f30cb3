"""Host-side phase costs of the bench's e2e step (public numpy API)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_1802_09113_b200 as snx
from paper_1802_09113_b200 import sampling
N, P, C = 50000, 3072, 10
A, y = oracle.synthetic_problem(N, P, C, seed=0)
prob = snx.SoftmaxProblem(snx.DeviceDataset.from_numpy(A, y, C), 1e-3)
x = 0.01 * np.random.default_rng(7).standard_normal((C - 1) * P)
g = np.random.default_rng(8).standard_normal((C - 1) * P)
cfg = snx.CgConfig(1e-4, 10)
sc = snx.SampleConfig(1.0, 0.05)
for k in range(5):
    snx.cg_solve(snx.SubsampledOracle(prob, sc, k).hessian_operator(x), g, cfg)
torch.cuda.synchronize()
T = {"draw": 0, "oracle": 0, "hessop": 0, "cg_solve": 0}
R = 50
for k in range(R):
    t0 = time.perf_counter()
    sampling._draw(sampling.stream_rng(0, 100 + k, 1), N, 2500, False)
    t1 = time.perf_counter()
    orc = snx.SubsampledOracle(prob, sc, 100 + k)
    t2 = time.perf_counter()
    op = orc.hessian_operator(x)
    t3 = time.perf_counter()
    snx.cg_solve(op, g, cfg)
    t4 = time.perf_counter()
    T["draw"] += t1 - t0; T["oracle"] += t2 - t1; T["hessop"] += t3 - t2; T["cg_solve"] += t4 - t3
print({k: round(v / R * 1e6, 1) for k, v in T.items()}, "us per step")
