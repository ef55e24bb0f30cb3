import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import load_golden
import paper_1802_09113_b200 as snx
from paper_1802_09113_b200 import _lib
cudart = ctypes.CDLL("libcudart.so.12") if False else None
orig = _lib.call
def traced(name, *args):
    st = torch.cuda.current_stream()
    cap = torch.cuda.is_current_stream_capturing()
    r = orig(name, *args)
    # query capture status of the current stream
    status = ctypes.c_int(-1)
    lib = ctypes.CDLL(None)
    print(f"{name:22s} capturing={cap} after={torch.cuda.is_current_stream_capturing()}", flush=True)
    return r
_lib.call = traced
g = load_golden("solver_golden.npz")
for i in range(5):
    k = f"nt{i}_"
    n, p, C, seed, lam, iters, sseed = g[k + "params"]
    ds = snx.DeviceDataset.from_numpy(g[k + "A"], g[k + "y"], int(C))
    cfg = snx.make_variant(str(g[k + "variant"]), snx.NewtonConfig(max_outer_iters=int(iters), samples=snx.SampleConfig(seed=int(sseed))))
    print("=== case", i, str(g[k + "variant"]), n, p, C, flush=True)
    try:
        tr = snx.newton_solve(snx.SoftmaxProblem(ds, float(lam)), cfg)
        print("ok", tr.reason, len(tr.records))
    except Exception as e:
        print("FAIL", type(e).__name__, str(e)[:200])
        break
