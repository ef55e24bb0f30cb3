import os, sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import oracle
import paper_1802_09113_b200 as snx
N, P, C = 50000, 3072, 10
A, y = oracle.synthetic_problem(N, P, C, seed=0)
ds = snx.DeviceDataset.from_numpy(A, y, C)
prob = snx.SoftmaxProblem(ds, 1e-3)
x = 0.01 * np.random.default_rng(7).standard_normal((C - 1) * P)
g = np.random.default_rng(8).standard_normal((C - 1) * P)
cfg = snx.CgConfig(1e-4, 10)
def step(k):
    orc = snx.SubsampledOracle(prob, snx.SampleConfig(1.0, 0.05), k)
    return snx.cg_solve(orc.hessian_operator(x), g, cfg).iterations
for k in range(5): step(k)
torch.cuda.synchronize()
import cProfile, pstats
t0 = time.perf_counter()
for k in range(50): step(100 + k)
dt = (time.perf_counter() - t0) / 50
print(f"e2e step {dt*1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
for k in range(50): step(200 + k)
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(25)
