"""BASELINE config #5 per GPU: one 1M x 3072 row shard of the 8M x 3072,
C = 100 problem (f32 data, 12.3 GB in HBM), 5% Hessian sample (m = 50k),
the wide tensor-core Hessian product and a 10-product CG solve.

    python tools/large_shard.py [n_rows] [reps] [solve_iters] [f32|f64]
"""
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_09113_b200 as snx  # noqa: E402
from paper_1802_09113_b200 import cg as cgmod, softmax  # noqa: E402

def measure(n=1_000_000, reps=10, p=3072, C=100, seed=0, solve_iters=0, dtype="f32"):
    """Prepare + Hessian product + 10-product CG on an n x p shard (device data):
    f32 on the wide tensor-core pair, or f64 on the wide fp64 path (library
    DGEMMs + row kernels, csrc/snx_wide64.cu)."""
    K = C - 1
    g = torch.Generator(device="cuda").manual_seed(seed)
    tdt = torch.float32 if dtype == "f32" else torch.float64
    X = torch.randn((n, p), generator=g, device="cuda", dtype=tdt)
    X.mul_(1.0 / math.sqrt(n))
    labels = torch.randint(0, C, (n,), generator=g, device="cuda", dtype=torch.int32)
    ds = snx.DeviceDataset(X, labels, C, p, dtype=dtype)
    x = 0.05 * torch.randn(K * p, generator=g, device="cuda", dtype=torch.float64)
    v = torch.randn(K * p, generator=g, device="cuda", dtype=torch.float64)
    view = ds.take(snx.draw_samples(snx.SampleConfig(1.0, 0.05), n, 0)[1])
    m = view.n_rows
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    op = softmax.HessianOperator(view, x, 1e-3, scale=n / m)  # warm-up prepare
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(3):
        op = softmax.HessianOperator(view, x, 1e-3, scale=n / m)
    e1.record(st)
    torch.cuda.synchronize()
    prep_ms = e0.elapsed_time(e1) / 3
    out = torch.empty_like(v)
    for _ in range(3):
        op.apply_into(v, out)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        op.apply_into(v, out)
    e1.record(st)
    torch.cuda.synchronize()
    hv_ms = e0.elapsed_time(e1) / reps
    for _ in range(2):
        ws = cgmod.cg_graph_for(op, 10, 1e-4).run(v)
    torch.cuda.synchronize()
    e0.record(st)
    ws = cgmod.cg_graph_for(op, 10, 1e-4).run(v)
    e1.record(st)
    torch.cuda.synchronize()
    cg_ms = e0.elapsed_time(e1)
    iters = int(ws.slot(10)[3])
    useful = 4.0 * m * p * K                 # 2 GEMMs x 2 m p K
    KP = (K + 15) // 16 * 16
    if dtype == "f32":
        issued = 2.0 * 2 * m * p * (3 * KP)  # per GEMM: N = 2 KP plus N = KP, bf16
        xbytes = 2 * 2 * m * p * 2           # X1 + X2 (bf16) read by each GEMM
    else:
        issued = useful                      # DGEMM: fp64 operands as they are
        xbytes = 2 * m * p * 8               # X_S read by each DGEMM
    solve = None
    if solve_iters:
        prob = snx.SoftmaxProblem(ds, 1e-3)
        cfg = snx.make_variant("subsampled-100", snx.NewtonConfig(max_outer_iters=solve_iters))
        snx.newton_solve(prob, snx.make_variant("subsampled-100",
                                                snx.NewtonConfig(max_outer_iters=1)))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tr = snx.newton_solve(prob, cfg)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        solve = {"outer_iters": tr.iterations, "seconds": dt, "ms_per_iter": 1e3 * dt /
                 max(tr.iterations, 1), "reason": tr.reason,
                 "objective": [r.objective for r in tr.records],
                 "cg_iters": [r.cg_iters for r in tr.records[1:]]}
    res = {
        "newton_solve": solve,
        "workload": (f"{n}x{p} f32 shard, C={C}, 5% S_H (m={m}), tcgen05 bf16 two-term split"
                     if dtype == "f32" else
                     f"{n}x{p} fp64 shard, C={C}, 5% S_H (m={m}), fp64 DGEMMs (cuBLAS) + "
                     "row kernels, the reference's precision"),
        "prepare_ms": prep_ms, "hess_apply_ms": hv_ms, "hv_per_s": 1e3 / hv_ms,
        "cg_10_ms": cg_ms, "cg_iters": iters, "cg_hv_per_s": iters / (cg_ms / 1e3),
        "useful_tflops": useful / (hv_ms / 1e3) / 1e12,
        "issued_mma_tflops": issued / (hv_ms / 1e3) / 1e12,
        "cg_graph_captured": cgmod.cg_graph_for(op, 10, 1e-4).graph is not cgmod._EAGER,
        "x_stream_tb_s": xbytes / (hv_ms / 1e3) / 1e12,
    }
    return res, op, v, out


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    solve_iters = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    res, op, v, out = measure(n, reps, solve_iters=solve_iters,
                              dtype=sys.argv[4] if len(sys.argv) > 4 else "f32")
    print(json.dumps(res))

if __name__ == "__main__" and os.environ.get("SNX_LIB", "").endswith("libsnx_tl.so"):
    import ctypes

    from paper_1802_09113_b200 import _lib

    op.apply_into(v, out)
    torch.cuda.synchronize()
    b = (ctypes.c_ulonglong * (2 * 160 * 8))()
    assert _lib.load().snx_debug_tc_timeline(b) == 0
    t = np.frombuffer(b, dtype=np.uint64).reshape(2, 160, 8).astype(np.int64)[:, :148]
    base = t[0, :, 0][t[0, :, 0] > 0].min()
    for k, nm in enumerate(["tcw_gemm1", "tcw_gemm2"]):
        for ev, en in enumerate(["entry", "1st data", "mma done", "exit", "V in smem",
                                 "row loop", "U stored", "epi end"]):
            col = t[k, :, ev]
            col = col[col > 0]
            if len(col) == 0:
                continue
            print(f"{nm} {en:9s} med {(np.median(col) - base) / 1e3:8.2f} max "
                  f"{(col.max() - base) / 1e3:8.2f} min {(col.min() - base) / 1e3:8.2f}")
