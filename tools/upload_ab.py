"""e2e bench step (numpy in / out through the public API) with the two upload
strategies of device.upload: pageable async copies vs a pinned allocation per call."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import oracle
import paper_1802_09113_b200 as snx
from paper_1802_09113_b200 import device
N, P, C = 50000, 3072, 10
A, y = oracle.synthetic_problem(N, P, C, seed=0)
ds = snx.DeviceDataset.from_numpy(A, y, C)
prob = snx.SoftmaxProblem(ds, 1e-3)
x = 0.01 * np.random.default_rng(7).standard_normal((C - 1) * P)
g = np.random.default_rng(8).standard_normal((C - 1) * P)
cfg = snx.CgConfig(1e-4, 10)
sc = snx.SampleConfig(1.0, 0.05)
def step(k):
    orc = snx.SubsampledOracle(prob, sc, k)
    return snx.cg_solve(orc.hessian_operator(x), g, cfg).iterations
def run(tag):
    for k in range(5): step(k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(50): step(100 + k)
    print(tag, round((time.perf_counter() - t0) / 50 * 1e6, 1), "us/step")
run("device.upload (pageable up to 4 MB)")
orig = device.upload
def pinned(a, dev=None):
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().to(dev or device.cuda_device(),
                                                                    non_blocking=True)
device.upload = pinned
run("pinned staging per call")
device.upload = orig
run("device.upload again")

# downloads: pinned buffers + one synchronisation (device.download) vs pageable .cpu()
orig_d = device.download


def pageable_download(*ts):
    torch.cuda.current_stream().synchronize()
    return [t.cpu().numpy() for t in ts]


device.download = pageable_download
run("download via pageable .cpu()")
device.download = orig_d
run("device.download (pinned)")
