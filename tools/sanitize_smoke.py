"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): every kernel family once -- fp64 / f32 row passes, the one-pass
kernels (column split with a 2-CTA cluster exchange, row split), the
tensor-core narrow and wide products, CG and Steihaug graphs, CSR, power step,
data prep."""
import os, sys
import numpy as np, torch, scipy.sparse as sp
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_1802_09113_b200 as snx
from paper_1802_09113_b200.sparse import CsrDataset
A, y = oracle.synthetic_problem(700, 200, 10, seed=1)
for dt in ("f64", "f32"):
    ds = snx.DeviceDataset.from_numpy(A, y, 10, dtype=dt)
    prob = snx.SoftmaxProblem(ds, 1e-3)
    tr = snx.newton_solve(prob, snx.make_variant("subsampled-100", snx.NewtonConfig(max_outer_iters=2)))
    snx.trust_region_solve(prob, snx.TrustRegionConfig(max_outer_iters=2))
    snx.class_probabilities(ds, tr.x_final)
# one-pass kernels: p = 900 -> 2-CTA clusters (DSMEM exchange), p = 54 -> row split;
# sampled Hessians gather through row indices, full gradients on both
for n3, p3, C3 in ((500, 900, 10), (3000, 54, 7)):
    A3, y3 = oracle.synthetic_problem(n3, p3, C3, seed=4)
    ds3 = snx.DeviceDataset.from_numpy(A3, y3, C3)
    snx.newton_solve(snx.SoftmaxProblem(ds3, 1e-3),
                     snx.make_variant("subsampled-100", snx.NewtonConfig(max_outer_iters=2)))
    snx.gradient(snx.SoftmaxProblem(ds3, 1e-3), np.zeros((C3 - 1) * p3))
A2, y2 = oracle.synthetic_problem(600, 64, 40, seed=2)
ds2 = snx.DeviceDataset.from_numpy(A2, y2, 40, dtype="f32")
snx.newton_solve(snx.SoftmaxProblem(ds2, 1e-3), snx.make_variant("subsampled-100", snx.NewtonConfig(max_outer_iters=1)))
rng = np.random.default_rng(3)
M = sp.random(400, 300, density=0.05, format="csr", random_state=3)
cs = CsrDataset.from_scipy(M, rng.integers(0, 5, 400), 5)
snx.newton_solve(snx.SoftmaxProblem(cs, 1e-3), snx.make_variant("subsampled-100", snx.NewtonConfig(max_outer_iters=2)))
snx.estimate_lipschitz(snx.SoftmaxProblem(snx.DeviceDataset.from_numpy(A, y, 10), 0.0), iters=3)
snx.normalize_columns(snx.DeviceDataset.from_numpy(A, y, 10))
torch.cuda.synchronize()
print("sanitize workload done")
