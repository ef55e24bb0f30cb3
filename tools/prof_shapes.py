"""Timing driver: fp64 Hessian product / full gradient / captured CG solve /
prepare at the BASELINE shapes (CUDA events, back-to-back launches).

    python tools/prof_shapes.py [cifar,mnist,covertype] [reps]
SNX_FRAC=1.0 samples the whole dataset (the full-Newton products).
SNX_TWO_PASS=1 selects the two-GEMM kernels (snx_rowpass.cu) for an A/B."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_09113_b200 as snx  # noqa: E402
from paper_1802_09113_b200 import cg as cgmod  # noqa: E402

SHAPES = {"cifar": (50000, 3072, 10), "mnist": (60000, 784, 10), "covertype": (581012, 54, 7)}


def timed(fn, reps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def persist_l2():
    """SNX_PERSIST=1: set aside the maximum persisting-L2 carve-out (what the
    kernels' evict_last bulk copies need to stay resident)."""
    import ctypes
    import glob
    torch.zeros(1, device="cuda")
    lib = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime",
                                 "lib", "libcudart.so.*"))[0]
    rt = ctypes.CDLL(lib)
    v = ctypes.c_int()
    rt.cudaDeviceGetAttribute(ctypes.byref(v), 108, 0)  # cudaDevAttrMaxPersistingL2CacheSize
    rc = rt.cudaDeviceSetLimit(6, ctypes.c_size_t(v.value))  # cudaLimitPersistingL2CacheSize
    print(f"persisting L2 carve-out {v.value / 2**20:.1f} MiB (rc {rc})")


def main():
    if os.environ.get("SNX_PERSIST"):
        persist_l2()
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else list(SHAPES)
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    tag = "two-pass" if os.environ.get("SNX_TWO_PASS") else "cluster"
    for name in names:
        n, p, C = SHAPES[name]
        gen = np.random.default_rng(0)
        A = gen.standard_normal((n, p))
        A /= np.sqrt((A ** 2).sum(axis=0))
        y = gen.integers(0, C, size=n)
        ds = snx.DeviceDataset.from_numpy(A, y, C)
        prob = snx.SoftmaxProblem(ds, 1e-3)
        x = torch.from_numpy(0.01 * np.random.default_rng(7).standard_normal((C - 1) * p)).cuda()
        frac = float(os.environ.get("SNX_FRAC", "0.05"))  # Hessian sample fraction
        orc = snx.SubsampledOracle(prob, snx.SampleConfig(1.0, frac), 0)
        g = orc.gradient_device(x)
        g = g[0] if isinstance(g, tuple) else g
        op = orc.hessian_operator(x)
        out = torch.empty_like(g)
        hv = timed(lambda: op.apply_into(g, out), reps)
        gr = timed(lambda: snx.softmax.gradient_parts(ds, x, 1.0, 1e-3), max(5, reps // 10))
        cgt = timed(lambda: cgmod.cg_graph_for(op, 10, 1e-4).run(g), max(5, reps // 5))
        prep = timed(lambda: op._prepare(), max(5, reps // 5))
        m = op.view.n_rows
        print(f"{tag} {name}: m={m} hess_apply {hv:.1f} us | full grad {gr:.1f} us | "
              f"cg_solve(10) {cgt:.1f} us | prepare {prep:.1f} us", flush=True)
        del ds, prob, op, orc
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
