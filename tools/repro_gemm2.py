import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch, oracle
import paper_1802_09113_b200 as snx
from paper_1802_09113_b200 import softmax
A, y = oracle.synthetic_problem(3001, 130, 5, seed=3001)
ds = snx.DeviceDataset.from_numpy(A, y, 5)
x = torch.from_numpy(0.1 * np.random.default_rng(1).standard_normal(4 * 130)).cuda()
view = ds.take(snx.draw_samples(snx.SampleConfig(1.0, 0.3), 3001, 0)[1])
op = softmax.HessianOperator(view, x, 1e-3, scale=3001 / view.n_rows)
v = torch.randn(520, dtype=torch.float64, device='cuda')
print(op.apply(v)[:3])
torch.cuda.synchronize()
print("ok")
