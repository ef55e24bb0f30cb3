"""GEMM1 / GEMM2 tail anatomy of one Hessian product inside the CG graph (debug
build): per CTA, atomic-arrival time and the end of the last-arriver epilogue."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_1802_09113_b200 as snx
from paper_1802_09113_b200 import _lib, cg as cgmod
A, y = oracle.synthetic_problem(50000, 3072, 10, seed=0)
ds = snx.DeviceDataset.from_numpy(A, y, 10)
x = torch.from_numpy(0.01 * np.random.default_rng(7).standard_normal(9 * 3072)).cuda()
orc = snx.SubsampledOracle(snx.SoftmaxProblem(ds, 1e-3), snx.SampleConfig(1.0, 0.05), 0)
g, _ = orc.gradient_device(x)
op = orc.hessian_operator(x)
for _ in range(3):
    cgmod.cg_graph_for(op, 10, 1e-4).run(g)
torch.cuda.synchronize()
lib = _lib.load()
b = (ctypes.c_ulonglong * (3 * 160 * 8))()
assert lib.snx_debug_timeline(b) == 0
t = np.frombuffer(b, dtype=np.uint64).reshape(3, 160, 8).astype(np.int64)[:, :148]
for k, nm in enumerate(["gemm1", "gemm2"]):
    tt = t[k]
    b0 = tt[:, 0].min()
    rel = lambda c: (c - b0) / 1e3
    valid = lambda c: c >= b0
    atom, ex, e0, e1, cd, sw = tt[:, 5], tt[:, 3], tt[:, 6], tt[:, 7], tt[:, 2], tt[:, 4]
    epi = np.where(valid(e1), e1, np.where(valid(e0), e0, 0))
    has = epi > 0
    print(f"{nm}: CTAs with an epilogue this launch: {has.sum()}")
    print(f"  compute done  med {np.median(rel(cd)):6.2f} max {rel(cd).max():6.2f}")
    print(f"  seg written   med {np.median(rel(sw)):6.2f} max {rel(sw).max():6.2f}")
    print(f"  atomic        med {np.median(rel(atom)):6.2f} max {rel(atom).max():6.2f}")
    if has.any():
        d = (epi[has] - atom[has]) / 1e3
        print(f"  epilogue end - own atomic: med {np.median(d):5.2f} max {d.max():5.2f} us;"
              f" epilogue end max {rel(epi[has]).max():6.2f}")
        dd = (ex[has] - epi[has]) / 1e3
        print(f"  exit - epilogue end (epilogue CTAs): med {np.median(dd):5.2f}")
    print(f"  exit          med {np.median(rel(ex)):6.2f} max {rel(ex).max():6.2f}")
