"""Benchmark: sub-sampled Hessian-vector products/s at CIFAR-10 shape
(BASELINE.json metric; configs[2]: 50k x 3072, C=10, 5% Hessian sample).

One step = one outer iteration's sampled-Hessian work on fresh inputs: the
step's S_H indices uploaded (pinned H2D inside the timed region), the Hessian
operator prepared on them (gather fused into the one-pass kernel) and a device
CG solve (theta=1e-4, <=10 Hessian products, reference cg.py), all device
resident.  value = Hessian products applied / device time.  Also reported:
e2e through the public numpy API (host buffers, H2D/D2H in the timed
region), the roofline of the Hessian product, the CG kernels' GB/s, a CPU
baseline (the oracle port on this host), time-to-tolerance per SURVEY 8(d)
(planted-softmax labels, eps = 1e-6 |grad F(0)|, 100-iteration cap, the CPU
port run to the same tolerance), the trust-region config #4, and the other
BASELINE shapes.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

With --gpus N > 1 and no torchrun environment the script re-launches itself
under torch.distributed.run with N ranks (one per GPU, NCCL); rows are then
sharded over the ranks (strong scaling of the CIFAR problem).
"""

import argparse
import json
import math
from dataclasses import replace
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N, P, C = 50000, 3072, 10
F_H, LAM, THETA, T_CG = 0.05, 1e-3, 1e-4, 10
METRIC = "subsampled Hessian-vector products/s (CIFAR-10 shape, 5% sample)"
UNIT = "Hv/s"
# the workload both arms run (printed identically by both)
CONFIG = {"workload": "cifar10-shape 50000x3072 C=10, 5% S_H (m=2500) per step: S_H gather + "
                      "h-prep + CG (theta=1e-4, <=10 Hv)",
          "n": N, "p": P, "C": C, "hessian_fraction": F_H, "lam": LAM, "theta": THETA,
          "cg_max_iters": T_CG, "data": "N(0,1) features, unit-norm columns, uniform labels",
          "l2": "inputs > L2: 1.23 GB X in HBM, fresh S_H gathered every step"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms by ONE
    background nvidia-smi process started before the timed region (no fork
    inside it); the summary keeps the samples taken while the region ran."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # first sample lands before the timed region
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.1)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=10)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out = ""
        self.samples = [[t.strip() for t in ln.split(",")] for ln in out.splitlines() if ln]

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(self.samples[0][1]) if self.samples else None,
                "reasons": reasons, "samples": len(self.samples)}


# dram__bytes_read.sum + dram__bytes_write.sum of one Hessian product (the
# one-pass kernel + its finalize), from the committed ncu --set full capture
# (per launch, cold cache); None until profiled
# main kernel dram read + write (r02b capture) + the finalize kernel's (r02 capture)
TRAFFIC = {"f64": 61.933568e6 + 1.92128e6 + 7.529984e6}
TRAFFIC_SOURCE = "profiles/r02b_onepass_ncu_full.txt (+ finalize_kernel: profiles/r02_onepass_ncu_full.txt)"
KERNEL_NAME = {"f64": "one-pass cluster row pass (cluster_rowpass_kernel<9> + finalize_kernel, "
                      "csrc/snx_cluster.cu)",
               "f32": "tcgen05 tc_gemm1 + tc_gemm2 (csrc/snx_tc.cu)"}


def synthetic_problem(n, p, nC, seed=0, normalize=True, ill_conditioned=False):
    """Synthetic data per SURVEY.md 8(d): N(0,1) features (numpy default_rng), columns
    scaled to unit norm (dataset.py:314-324) or, for the trust-region config, by
    logspace(2, -4, p) (tests/test_acceptance.py:223-229); uniform labels.  The same
    recipe as the tests' fixtures, kept here so the measured legs do not import
    the oracle (which only the CPU-baseline legs run)."""
    gen = np.random.default_rng(seed)
    A = gen.standard_normal((n, p))
    y = gen.integers(0, nC, size=n).astype(np.int64)
    if ill_conditioned:
        A *= np.logspace(2, -4, p)
    elif normalize:
        norms = np.sqrt((A ** 2).sum(axis=0))
        A *= np.where(norms > 0, 1.0 / np.where(norms > 0, norms, 1.0), 1.0)
    return np.ascontiguousarray(A), y


def make_problem(seed=0):
    return synthetic_problem(N, P, C, seed=seed)


def cpu_baseline(A, y, x, steps_budget_s=10.0, max_steps=1000):
    """The oracle port (numpy/OpenBLAS fp64) on the same step: h-prep on a fresh
    S_H + CG with <= 10 Hessian products; bounded to ~steps_budget_s."""
    import oracle

    g = oracle.grad(A, y, C, x, LAM)
    hv, t_total, steps = 0, 0.0, 0
    while steps < max_steps and t_total < steps_budget_s:
        s_h = oracle.draw_samples(1.0, F_H, False, 0, N, 1000 + steps)[1]
        t0 = time.perf_counter()
        Ah, yh = A[s_h], y[s_h]
        h = oracle.hess_probs(Ah, yh, C, x)
        count = [0]

        def op(v):
            count[0] += 1
            return oracle.hess_apply(Ah, h, C, v, N / len(s_h), LAM)

        oracle.cg(op, g, THETA, T_CG)
        t_total += time.perf_counter() - t0
        hv += count[0]
        steps += 1
    return {"value": hv / t_total, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": f"{steps} steps (S_H gather + h-prep + CG, {hv} Hv) of the CIFAR-shape "
                      f"workload, numpy/OpenBLAS fp64, {t_total:.1f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    A, y = make_problem()
    x = 0.01 * np.random.default_rng(7).standard_normal((C - 1) * P)
    import oracle

    g = oracle.grad(A, y, C, x, LAM)
    for w in range(args.warmup):
        s_h = oracle.draw_samples(1.0, F_H, False, 0, N, w)[1]
        h = oracle.hess_probs(A[s_h], y[s_h], C, x)
        oracle.hess_apply(A[s_h], h, C, g, N / len(s_h), LAM)
    hv, t = 0, 0.0
    for k in range(args.steps):
        s_h = oracle.draw_samples(1.0, F_H, False, 0, N, 100 + k)[1]
        t0 = time.perf_counter()
        Ah, yh = A[s_h], y[s_h]
        h = oracle.hess_probs(Ah, yh, C, x)
        cnt = [0]

        def op(v):
            cnt[0] += 1
            return oracle.hess_apply(Ah, h, C, v, N / len(s_h), LAM)

        oracle.cg(op, g, THETA, T_CG)
        t += time.perf_counter() - t0
        hv += cnt[0]
    v = hv / t
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": CONFIG,
        "parallelism": f"host CPU, {os.cpu_count()} threads (numpy/OpenBLAS), rank 0 only",
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                         "sample": f"{args.steps} steps, oracle port (numpy/OpenBLAS fp64)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def shape_rate(snx, torch, A, y, nC, dtype, steps=30, warmup=3, frac=F_H):
    """Hv/s of the bench step (fresh S_H prepare + captured CG solve) at another
    BASELINE shape; device-timed with CUDA events."""
    from paper_1802_09113_b200 import cg as cgmod, softmax

    n, p = A.shape
    ds = snx.DeviceDataset.from_numpy(A, y, nC, dtype=dtype)
    x = torch.from_numpy(0.01 * np.random.default_rng(7).standard_normal((nC - 1) * p)).cuda()
    g, _ = softmax.gradient_parts(ds, x, 1.0, LAM)
    views = [ds.take(snx.draw_samples(snx.SampleConfig(1.0, frac), n, k)[1])
             for k in range(warmup + steps)]
    m = views[0].n_rows
    iters = torch.zeros(warmup + steps, dtype=torch.float64, device="cuda")
    keep = [None]

    def step(k):
        op = softmax.HessianOperator(views[k], x, LAM, scale=n / m)
        keep[0] = op
        ws = cgmod.cg_graph_for(op, T_CG, THETA).run(g)
        iters[k:k + 1].copy_(ws.slot(T_CG)[3:4])

    for k in range(warmup):
        step(k)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for k in range(warmup, warmup + steps):
        step(k)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    hv = int(iters[warmup:].sum())
    out = torch.empty_like(g)
    op = keep[0]
    for _ in range(3):
        op.apply_into(g, out)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(20):
        op.apply_into(g, out)
    e1.record(st)
    torch.cuda.synchronize()
    res = {"value": hv / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / steps, "steps": steps,
           "m": m, "dtype": dtype, "hess_apply_us": e0.elapsed_time(e1) / 20 * 1e3}
    del ds, views, keep, op
    torch.cuda.empty_cache()
    return res


def sparse_problem(n=11314, p=61188, nC=20, density=0.0023, seed=0):
    import scipy.sparse as sp

    rng = np.random.default_rng(seed)
    A = sp.random(n, p, density=density, format="csr", random_state=seed,
                  data_rvs=lambda k: rng.uniform(0.0, 1.0, k))
    norms = np.sqrt(np.asarray(A.multiply(A).sum(axis=0)).ravel())
    scale = np.where(norms > 0, 1.0 / np.where(norms > 0, norms, 1.0), 1.0)
    A = sp.csr_array(A @ sp.diags(scale))
    y = rng.integers(0, nC, n)
    return A, y


def sparse_rate(snx, torch, steps=30, warmup=3):
    """Hv/s of the bench step on CSR data (fresh S_H gather + prepare + captured
    CG), device-timed; the oracle port on scipy CSR (the reference's sparse
    arithmetic) timed on the host for comparison."""
    import oracle
    from paper_1802_09113_b200 import cg as cgmod, softmax
    from paper_1802_09113_b200.sparse import CsrDataset

    A, y = sparse_problem()
    n, p = A.shape
    nC = 20
    ds = CsrDataset.from_scipy(A, y, nC)
    x = torch.from_numpy(0.01 * np.random.default_rng(7).standard_normal((nC - 1) * p)).cuda()
    g, _ = softmax.gradient_parts(ds, x, 1.0, LAM)
    views = [ds.take(snx.draw_samples(snx.SampleConfig(1.0, F_H), n, k)[1])
             for k in range(warmup + steps)]
    m = views[0].n_rows
    iters = torch.zeros(warmup + steps, dtype=torch.float64, device="cuda")
    keep = [None]

    def step(k):
        op = softmax.HessianOperator(views[k], x, LAM, scale=n / m)
        keep[0] = op
        ws = cgmod.cg_graph_for(op, T_CG, THETA).run(g)
        iters[k:k + 1].copy_(ws.slot(T_CG)[3:4])

    for k in range(warmup):
        step(k)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for k in range(warmup, warmup + steps):
        step(k)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    hv = int(iters[warmup:].sum())
    op, out_v = keep[0], torch.empty_like(g)
    for _ in range(3):
        op.apply_into(g, out_v)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(50):
        op.apply_into(g, out_v)
    e1.record(st)
    torch.cuda.synchronize()
    apply_us = e0.elapsed_time(e1) / 50 * 1e3
    for _ in range(3):
        softmax.gradient_parts(ds, x, 1.0, LAM)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(20):
        softmax.gradient_parts(ds, x, 1.0, LAM)
    e1.record(st)
    torch.cuda.synchronize()
    grad_us = e0.elapsed_time(e1) / 20 * 1e3
    # CPU: the oracle port on scipy CSR, same step (bounded sample)
    xh = x.cpu().numpy()
    gh = g.cpu().numpy()
    t0, cnt, steps_cpu = time.perf_counter(), 0, 0
    while time.perf_counter() - t0 < 5.0 and steps_cpu < 50:
        s_h = oracle.draw_samples(1.0, F_H, False, 0, n, 900 + steps_cpu)[1]
        As, ys = A[s_h], y[s_h]
        h = oracle.hess_probs(As, ys, nC, xh)
        c = [0]

        def opc(v):
            c[0] += 1
            return oracle.hess_apply(As, h, nC, v, n / len(s_h), LAM)

        oracle.cg(opc, gh, THETA, T_CG)
        cnt += c[0]
        steps_cpu += 1
    cpu_s = time.perf_counter() - t0
    nnz_s = int(views[-1].base.sample_nnz(views[-1].idx))
    return {"value": hv / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / steps, "m": m,
            "nnz": int(A.nnz), "sample_nnz": nnz_s, "hess_apply_us": apply_us,
            "full_gradient_us": grad_us,
            "cpu_port_hv_per_s": cnt / cpu_s, "cpu_cores": os.cpu_count(),
            "workload": f"newsgroups20-shape CSR {n}x{p} C={nC}, nnz {A.nnz}, 5% S_H, fp64"}


def secondary(snx, torch, args):
    """The other BASELINE.json shapes and the tensor-core f32 path (one GPU)."""
    import oracle

    out = {}
    for name, n, p, nC in (("mnist", 60000, 784, 10), ("covertype", 581012, 54, 7)):
        A, y = synthetic_problem(n, p, nC, seed=0)
        out[name] = shape_rate(snx, torch, A, y, nC, "f64")
        out[name]["workload"] = f"{name}-shape {n}x{p} C={nC}, 5% S_H, fp64"
        del A, y
    if args.dtype == "f64":
        from paper_1802_09113_b200 import device as snx_device

        A, y = make_problem()
        out["cifar10_f32"] = shape_rate(snx, torch, A, y, C, "f32")
        out["cifar10_f32"]["workload"] = (
            "cifar10-shape, f32 data: the one-pass kernel on f32 rows widened to fp64 "
            "(half the bytes of X_S, fp64 arithmetic)")
        snx_device.F32_TENSOR_CORES = True  # the tcgen05 pair on the same data, for comparison
        out["cifar10_f32_tensor_core"] = shape_rate(snx, torch, A, y, C, "f32")
        out["cifar10_f32_tensor_core"]["workload"] = (
            "cifar10-shape, f32 data, Hessian GEMMs on tcgen05 (bf16 two-term split), 1e-4 path")
        snx_device.F32_TENSOR_CORES = False
    # estimate_lipschitz (bench.py:116-138 of the reference): 200 power
    # iterations of the full-data (50k x 3072) Hessian product at x = 0
    A, y = make_problem()
    ds = snx.DeviceDataset.from_numpy(A, y, C)
    lprob = snx.SoftmaxProblem(ds, LAM)
    snx.estimate_lipschitz(lprob, iters=3)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    L = snx.estimate_lipschitz(lprob, iters=200)
    dt = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.estimate_lipschitz(A, y, C, iters=5)
    cpu5 = time.perf_counter() - t0
    full_bytes = N * P * 8  # X streamed once per product (the one-pass row pass)
    out["lipschitz_cifar10"] = {
        "seconds": dt, "iters": 200, "L": L, "ms_per_iter": dt / 200 * 1e3,
        "x_stream_gb_s": full_bytes / (dt / 200) / 1e9,
        "cpu_port_seconds_extrapolated": cpu5 / 5 * 200, "cpu_cores": os.cpu_count(),
        "workload": "cifar10-shape full-data Hessian power iteration at x=0, lam=0, fp64"}
    del ds, lprob, A, y
    torch.cuda.empty_cache()
    # CSR storage (the paper's Newsgroups20 / cuSPARSE path): 11314 x
    # 61188, C = 20, ~1.6M nonzeros, columns normalised; fresh 5% S_H + CG per step
    out["newsgroups20_sparse"] = sparse_rate(snx, torch)
    torch.cuda.empty_cache()
    # BASELINE config #5 per GPU: a 1M x 3072 f32 shard of the 8M x 3072, C = 100
    # problem (row-sharded over 8 GPUs; one GPU here), wide tensor-core product
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import large_shard

    res, _, _, _ = large_shard.measure(1_000_000, 10, solve_iters=5)
    out["large_c100_shard_f32"] = res
    torch.cuda.empty_cache()
    # the same shard in fp64 (the reference's precision): library DGEMMs + row
    # kernels (csrc/snx_wide64.cu)
    res, _, _, _ = large_shard.measure(1_000_000, 10, solve_iters=3, dtype="f64")
    out["large_c100_shard_f64"] = res
    torch.cuda.empty_cache()
    return out


def planted_problem(n, p, nC, seed=0, scale=3.0):
    """Planted-softmax labels (SURVEY 8(d) time-to-tolerance): unit-norm N(0,1)
    columns, labels drawn from softmax(A W*) with W* ~ scale * N(0,1), so the
    regularised solve has a meaningful optimum (tools/tol_probe.py)."""
    gen = np.random.default_rng(seed)
    A = gen.standard_normal((n, p))
    A /= np.sqrt((A ** 2).sum(axis=0))
    W = gen.standard_normal((p, nC)) * scale
    Z = A @ W
    Z -= Z.max(axis=1, keepdims=True)
    Pr = np.exp(Z)
    Pr /= Pr.sum(axis=1, keepdims=True)
    u = gen.random(n)[:, None]
    y = (Pr.cumsum(axis=1) < u).sum(axis=1).clip(0, nC - 1)
    return np.ascontiguousarray(A), y.astype(np.int64)


def time_to_tolerance(snx, torch, rank, world, skip_cpu):
    """SURVEY 8(d) metric 2: newton_solve from x0 = 0 until |grad| < 1e-6 |grad F(0)|
    (100-iteration cap) on planted labels at CIFAR shape, the reference's timed
    region (newton.py:72-104: objective / accuracy passes included); the oracle
    port runs the same solve on the host (all threads, and a 1-thread sample)."""
    from paper_1802_09113_b200 import softmax
    from paper_1802_09113_b200.device import dot

    A, y = planted_problem(N, P, C)
    ds = snx.DeviceDataset.from_numpy(A, y, C)
    prob = snx.SoftmaxProblem(ds, LAM)
    x0 = torch.zeros((C - 1) * P, dtype=torch.float64, device="cuda")
    gz = softmax.gradient_parts(ds, x0, 1.0, LAM)[0]
    g0 = math.sqrt(float(dot(gz, gz)))
    eps = 1e-6 * g0
    out = {"workload": "cifar10-shape 50000x3072 C=10, planted-softmax labels (scale 3), "
                       "lam=1e-3, x0=0", "epsilon": eps, "epsilon_rel_to_grad0": 1e-6,
           "max_outer_iters": 100}
    for name, variant in (("subsampled_100", "subsampled-100"), ("full_newton", "full")):
        ncfg = snx.make_variant(variant, snx.NewtonConfig(epsilon=eps, max_outer_iters=100))
        # warm-up: one outer iteration captures this variant's CUDA graphs
        snx.newton_solve(prob, replace(ncfg, max_outer_iters=1), x0=x0.clone())
        torch.cuda.synchronize()
        runs = []
        for _ in range(3):  # the same deterministic solve three times: best of 3
            t0 = time.perf_counter()
            tr = snx.newton_solve(prob, ncfg, x0=x0.clone())
            torch.cuda.synchronize()
            runs.append(time.perf_counter() - t0)
        dt = min(runs)
        out[name] = {"time_to_tol_s": dt, "runs_s": runs, "outer_iters": tr.iterations,
                     "ms_per_outer_iter": 1e3 * dt / max(tr.iterations, 1), "reason": tr.reason,
                     "final_objective": tr.final_objective,
                     "cg_iters": [r.cg_iters for r in tr.records[1:]],
                     "alphas": sorted({r.step_size for r in tr.records[1:]})}
    del ds, prob
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not skip_cpu:
        import oracle
        from threadpoolctl import threadpool_limits

        cpu = {"cores": os.cpu_count(), "kind": "port",
               "note": "oracle port (numpy/OpenBLAS fp64, the reference's arithmetic) on this "
                       "host, same problem, same epsilon and cap"}
        for name, variant in (("subsampled_100", "subsampled-100"), ("full_newton", "full")):
            t0 = time.perf_counter()
            ref = oracle.newton_solve(A, y, C, LAM, variant, epsilon=eps, max_outer_iters=100)
            dt = time.perf_counter() - t0
            it = len(ref["records"]) - 1
            cpu[name] = {"time_to_tol_s": dt, "outer_iters": it, "reason": ref["reason"],
                         "final_objective": ref["records"][-1][1],
                         "gpu_speedup": dt / out[name]["time_to_tol_s"]}
            with threadpool_limits(limits=1):  # 1-thread row: a 2-iteration sample
                t0 = time.perf_counter()
                oracle.newton_solve(A, y, C, LAM, variant, epsilon=eps, max_outer_iters=2)
                per = (time.perf_counter() - t0) / 2
            cpu[name]["one_thread_s_per_outer_iter"] = per
            cpu[name]["one_thread_time_to_tol_s_extrapolated"] = per * it
        out["cpu_port"] = cpu
    return out


def trust_region_config4(snx, torch, rank, world, skip_cpu):
    """BASELINE config #4: TR Steihaug-CG, ill-conditioned CIFAR shape
    (logspace(2,-4,p) columns), 10% S_H, eps = 1e-6 |grad F(0)|, 100-iteration
    cap; the CPU restatement (oracle/trust_region.py) timed on a bounded sample."""
    from paper_1802_09113_b200 import softmax
    from paper_1802_09113_b200.device import dot

    A, y = synthetic_problem(N, P, C, seed=0, normalize=False, ill_conditioned=True)
    ds = snx.DeviceDataset.from_numpy(A, y, C)
    prob = snx.SoftmaxProblem(ds, LAM)
    x0 = torch.zeros((C - 1) * P, dtype=torch.float64, device="cuda")
    gz = softmax.gradient_parts(ds, x0, 1.0, LAM)[0]
    eps = 1e-6 * math.sqrt(float(dot(gz, gz)))
    cfg = snx.TrustRegionConfig(epsilon=eps, max_outer_iters=100)
    snx.trust_region_solve(prob, snx.TrustRegionConfig(max_outer_iters=2))  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr = snx.trust_region_solve(prob, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    res = {"time_to_tol_s": dt, "outer_iters": tr.iterations, "reason": tr.reason,
           "ms_per_outer_iter": 1e3 * dt / max(tr.iterations, 1),
           "final_objective": tr.final_objective, "epsilon": eps, "hessian_fraction": 0.1,
           "workload": "cifar10-shape ill-conditioned (logspace(2,-4,p) columns), TR "
                       "Steihaug-CG, eps = 1e-6 |grad F(0)|, <= 100 outer iterations"}
    del ds, prob
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not skip_cpu:
        import oracle

        k = 3
        t0 = time.perf_counter()
        oracle.trust_region_solve(A, y, C, LAM, oracle.TrustRegionConfig(
            epsilon=eps, max_outer_iters=k), hessian_fraction=0.1)
        per = (time.perf_counter() - t0) / k
        res["cpu_port"] = {"s_per_outer_iter": per, "sample_outer_iters": k,
                           "time_to_tol_s_extrapolated": per * tr.iterations,
                           "cores": os.cpu_count(), "kind": "port (restatement; parity unpinned)"}
    return res


def sharded_extras(snx, torch, rank, world, dev, with_c100=True):
    """The N > 1 extras: newton_solve_sharded time-to-tolerance on
    the planted CIFAR-shape problem (rows sharded over the ranks: strong
    scaling), and BASELINE config #5 -- 1M x 3072 f32 rows per rank, C = 100,
    the wide tensor-core product -- as sharded Hessian products, a 10-product
    CG solve and outer iterations (weak scaling: per-rank rows fixed).  Times
    are the max over ranks."""
    import torch.distributed as dist

    from paper_1802_09113_b200 import cg as cgmod, distributed as sd

    def tmax(v):
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    out = {}
    # ---- time to tolerance, newton_solve_sharded (planted labels, eps = 1e-6 |grad F(0)|)
    A, y = planted_problem(N, P, C)
    sp = sd.ShardedProblem.from_global(A, y, C, LAM)
    del A, y
    x0 = torch.zeros(sp.dim, dtype=torch.float64, device=dev)
    g0 = sd.ShardedOracle(sp, snx.SampleConfig(1.0, 1.0), 0).gradient_device(x0)
    eps = 1e-6 * math.sqrt(float(torch.dot(g0, g0)))
    ncfg = snx.make_variant("subsampled-100", snx.NewtonConfig(epsilon=eps, max_outer_iters=100))
    sd.newton_solve_sharded(sp, replace(ncfg, max_outer_iters=1), x0=x0.clone())  # warm-up
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    tr = sd.newton_solve_sharded(sp, ncfg, x0=x0.clone())
    torch.cuda.synchronize()
    dt = tmax(time.perf_counter() - t0)
    out["time_to_tolerance_sharded"] = {
        "workload": f"cifar10-shape 50000x3072 C=10 planted labels, rows sharded over {world} "
                    "rank(s), newton_solve_sharded subsampled-100, eps = 1e-6 |grad F(0)|, <= 100 "
                    "outer iterations", "scaling": "strong", "epsilon": eps,
        "time_to_tol_s": dt, "outer_iters": tr.iterations, "reason": tr.reason,
        "ms_per_outer_iter": 1e3 * dt / max(tr.iterations, 1),
        "final_objective": tr.final_objective}
    del sp, x0, g0
    torch.cuda.empty_cache()
    if not with_c100:
        return out
    # ---- BASELINE config #5: 1M x 3072 f32 rows per rank, C = 100
    n_loc, p5, c5 = 1_000_000, 3072, 100
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    X = torch.randn((n_loc, p5), generator=gen, device=dev, dtype=torch.float32)
    X.mul_(1.0 / math.sqrt(n_loc * world))
    labels = torch.randint(0, c5, (n_loc,), generator=gen, device=dev, dtype=torch.int32)
    local = snx.DeviceDataset(X, labels, c5, p5, dtype="f32")
    sp5 = sd.ShardedProblem(local, n_loc * world, n_loc * rank, LAM)
    gx = torch.Generator(device=dev).manual_seed(7)  # the same x on every rank
    x = 0.05 * torch.randn(sp5.dim, generator=gx, device=dev, dtype=torch.float64)
    samples = snx.SampleConfig(1.0, F_H)
    g = sd.ShardedOracle(sp5, samples, 0).gradient_device(x)
    cgws = cgmod.CgWorkspace(sp5.dim, T_CG, dev)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def cg_step(k):
        op = sd.ShardedOracle(sp5, samples, k).hessian_operator(x)
        cgmod.enqueue_cg(op, g, THETA, T_CG, cgws)
        return op

    for k in range(2):
        op = cg_step(k)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    steps = 3
    e0.record(st)
    hv = 0
    for k in range(2, 2 + steps):
        op = cg_step(k)
        hv += int(cgws.slot(T_CG)[3])
    e1.record(st)
    torch.cuda.synchronize()
    ms = tmax(e0.elapsed_time(e1))
    v = g.clone()
    o = torch.empty_like(v)
    for _ in range(2):
        op.apply_into(v, o)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(5):
        op.apply_into(v, o)
    e1.record(st)
    torch.cuda.synchronize()
    hv_ms = tmax(e0.elapsed_time(e1) / 5)
    ncfg5 = snx.make_variant("subsampled-100", snx.NewtonConfig(max_outer_iters=3))
    sd.newton_solve_sharded(sp5, replace(ncfg5, max_outer_iters=1))  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr5 = sd.newton_solve_sharded(sp5, ncfg5)
    torch.cuda.synchronize()
    dt5 = tmax(time.perf_counter() - t0)
    out["config5_sharded"] = {
        "workload": f"BASELINE config #5: {n_loc} x {p5} f32 rows per rank ({n_loc * world} "
                    f"global), C = {c5}, 5% S_H, tensor-core (bf16 two-term split) products, "
                    "one all-reduce per product", "scaling": "weak",
        "hv_per_s": hv / (ms / 1e3), "ms_per_cg_step": ms / steps, "cg_products": hv,
        "hess_apply_ms": hv_ms,
        "newton": {"outer_iters": tr5.iterations, "seconds": dt5,
                   "ms_per_outer_iter": 1e3 * dt5 / max(tr5.iterations, 1),
                   "reason": tr5.reason, "objective": [r.objective for r in tr5.records]}}
    del X, labels, local, sp5, op, cgws
    torch.cuda.empty_cache()
    return out


def cg_kernel_rate(torch, ws, d, reps=50):
    """Achieved GB/s of the CG vector kernels (snx_cg_update = cg_step1 + cg_step2,
    cg.py:77-96): d-vector bytes per update (step1 reads p s r Hs, writes p r;
    step2 reads r s p, writes s pb) over their CUDA-event time."""
    from paper_1802_09113_b200 import _lib
    from paper_1802_09113_b200.device import ptr, stream_handle

    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    state = ws.state.clone()
    state[2::_lib.CG_SLOT] = 0.0  # clear the done flags: every update does its work

    def upd():
        _lib.call("snx_cg_update", 0, ws.T, d, ptr(ws.Hs), ptr(ws.dots), ptr(ws.r), ptr(ws.s),
                  ptr(ws.p), ptr(ws.pb), ptr(state), stream_handle())

    # the updates captured in a CUDA graph (as in the CG solve): kernel time,
    # not the host's ctypes launch rate
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(3):
            upd()
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for _ in range(reps):
            upd()
    graph.replay()
    torch.cuda.synchronize()
    e0.record(st)
    graph.replay()
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    nbytes = 11 * d * 8
    return {"us_per_update": us, "bytes_per_update": nbytes,
            "achieved_gb_s": nbytes / (us * 1e-6) / 1e9,
            "note": "graph-replayed; latency-bound at d = 27648 (2 kernels of 256 fixed "
                    "blocks, SURVEY 8(d)): the 2.4 MB move in well under a microsecond at HBM "
                    "speed"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1802_09113_b200 as snx
    from paper_1802_09113_b200 import cg as cgmod, softmax

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if os.environ.get("SNX_BENCH_ONE_DEVICE") == "1":
        local = 0  # smoke test of the N-rank path on a one-GPU box (with SNX_BENCH_BACKEND=gloo)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group(os.environ.get("SNX_BENCH_BACKEND", "nccl"))
    # the row-sharded code path (one all-reduce per product); SNX_BENCH_SHARDED=1
    # runs it at world size 1 too (all-reduce = identity) to exercise it on one GPU
    sharded = world > 1 or os.environ.get("SNX_BENCH_SHARDED") == "1"

    A, y = make_problem()
    x_host = 0.01 * np.random.default_rng(7).standard_normal((C - 1) * P)
    dev = torch.device("cuda", local)
    x = torch.from_numpy(x_host).to(dev)
    total = args.warmup + args.steps
    samples = snx.SampleConfig(1.0, F_H)
    iters = torch.zeros(total, dtype=torch.float64, device=dev)
    # each step's S_H is drawn on the host up front (numpy, as the reference);
    # its upload to the device happens inside the step (timed)
    s_h = [snx.draw_samples(samples, N, k)[1] for k in range(total)]
    if not sharded:
        ds = snx.DeviceDataset.from_numpy(A, y, C, dtype=args.dtype)
        prob = snx.SoftmaxProblem(ds, LAM)
        g, _ = softmax.gradient_parts(ds, x, 1.0, LAM)
        m = len(s_h[0])
        ops = [None]

        def step(k):
            view = ds.take(s_h[k])  # pinned H2D copy of the indices
            op = softmax.HessianOperator(view, x, LAM, scale=N / m)
            ops[0] = op  # keep only the latest operator alive
            ws = cgmod.cg_graph_for(op, T_CG, THETA).run(g)  # CUDA-graph replay of the CG loop
            iters[k:k + 1].copy_(ws.slot(T_CG)[3:4])
    else:
        # rows sharded over the ranks (strong scaling: the CIFAR problem is fixed)
        from paper_1802_09113_b200 import distributed as sd

        sp = sd.ShardedProblem.from_global(A, y, C, LAM, dtype=args.dtype)
        ds = sp.local
        prob = None
        g = sd.ShardedOracle(sp, samples, 0).gradient_device(x)
        m = len(s_h[0])
        cgws = cgmod.CgWorkspace(ds.dim, T_CG, dev)
        ops = [None]

        def step(k):
            op = sd.ShardedOracle(sp, samples, k).hessian_operator(x)
            ops[0] = op
            cgmod.enqueue_cg(op, g, THETA, T_CG, cgws)
            iters[k:k + 1].copy_(cgws.slot(T_CG)[3:4])

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(st)
        h0 = time.perf_counter()
        for k in range(args.warmup, total):
            step(k)
        host_ms = (time.perf_counter() - h0) * 1e3
        e1.record(st)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t)
    hv_count = int(iters[args.warmup:].sum())
    value = hv_count / (ms / 1e3)

    # ---- roofline of the dominant op: one Hessian product
    op = ops[0]
    v = g.clone()
    out = torch.empty_like(v)
    if sharded:
        op = op.op  # the local product (the all-reduce is timed in `value`)
    reps = 50
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(5):
        op.apply_into(v, out)
    torch.cuda.synchronize()
    ev[0].record(st)
    for _ in range(reps):
        op.apply_into(v, out)
    ev[1].record(st)
    torch.cuda.synchronize()
    hv_ms = ev[0].elapsed_time(ev[1]) / reps
    tb = 8 if args.dtype == "f64" else 4
    m_loc = op.view.n_rows  # rows this GPU streams per product
    alg_bytes = m_loc * P * tb + m_loc * (C - 1) * tb + 2 * ds.dim * 8
    pk, pk_kind = peaks()
    achieved = alg_bytes / (hv_ms / 1e3) / 1e9
    flops = 4 * m_loc * P * (C - 1)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "traffic": TRAFFIC.get(args.dtype),
                "traffic_source": TRAFFIC_SOURCE,
                "kernel": KERNEL_NAME.get(args.dtype), "peak_kind": pk_kind,
                "ms_per_launch": hv_ms, "bytes_per_launch": alg_bytes,
                "flops_per_launch": flops,
                "note": "algorithmic bytes: X_S read once + h + v + Hv (SURVEY 8(d)); in the "
                        "CG loop the sample rows are re-read from L2/HBM every product",
                # the same launch against the ceiling it is closest to: the fp64
                # tensor / FMA pipe (36.5 TFLOP/s measured, profiles/r02_fp64_pipe.txt)
                "alt_bounds": {"fp64_tflops": flops / (hv_ms / 1e3) / 1e12,
                               "fp64_peak_tflops": 36.5,
                               "fp64_frac": flops / (hv_ms / 1e3) / 1e12 / 36.5},
                # tensor-pipe utilisation of the product's MMAs from the committed ncu
                # captures (north star (b)): the fp64 tensor path (DMMA) of the headline
                # product, and the tcgen05 bf16 pipe of the declared f32 path (C = 10:
                # N = 9 columns, memory-bound by construction; C = 100: config #5)
                "tensor_pipe": {
                    "fp64_dmma_ops_pct_of_peak_elapsed": 26.8,
                    "fp64_dmma_cycles_active_pct": 36.1,
                    "source_fp64": "profiles/r02b_onepass_ncu_full.txt (cluster_rowpass_kernel<9>)",
                    "tcgen05_c10_pct_elapsed": [1.7, 2.0],
                    "source_c10": "profiles/r02_tc_ncu_full.txt (tc_gemm1 / tc_gemm2)",
                    "tcgen05_c100_pct_active": [23.0, 31.0],
                    "source_c100": "profiles/r01_tcw_large_shard_ncu_full.txt (tcw_gemm1 / 2)"}}
    cg_rate = None
    if not sharded:
        wsx = cgmod.cg_graph_for(ops[0], T_CG, THETA).ws
        cg_rate = cg_kernel_rate(torch, wsx, ds.dim)

    # ---- e2e: the public numpy API, host buffers in and out
    g_host = g.cpu().numpy()
    cfg = snx.CgConfig(THETA, T_CG)
    e2e_steps = max(10, min(args.steps, 50))

    def e2e_step(k):
        if not sharded:
            orc = snx.SubsampledOracle(prob, snx.SampleConfig(1.0, F_H), k)
        else:
            orc = sd.ShardedOracle(sp, snx.SampleConfig(1.0, F_H), k)
        return snx.cg_solve(orc.hessian_operator(x_host), g_host, cfg).iterations

    for k in range(3):  # warm-up (graph capture, pinned-buffer pools)
        e2e_step(400 + k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_hv = 0
    for k in range(e2e_steps):
        e2e_hv += e2e_step(500 + k)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t)
    e2e = {"value": e2e_hv / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": 2 * ds.dim * 8 + m * 8,
           "d2h_bytes_per_step": ds.dim * 8 + 8 * 8,
           "note": "public numpy API: SubsampledOracle + hessian_operator + cg_solve per step"}

    solve = tr4 = None
    if not sharded and not args.skip_solve:
        del A, y
        solve = time_to_tolerance(snx, torch, rank, world, args.skip_cpu)
        tr4 = trust_region_config4(snx, torch, rank, world, args.skip_cpu)
        A, y = make_problem()
    cpu = cpu_baseline(A, y, x_host) if (rank == 0 and world == 1 and not args.skip_cpu) \
        else None
    shapes = extras = None
    if world == 1 and not args.skip_shapes:
        del A, y
        shapes = secondary(snx, torch, args)
    if sharded and not args.skip_solve:
        extras = sharded_extras(snx, torch, rank, world, dev, with_c100=not args.skip_shapes)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "host_ms_per_step": host_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": args.dtype, "data": "synthetic", "config": CONFIG,
            "parallelism": (f"rows sharded over {world} GPU(s), one all-reduce per Hv"
                            if sharded else "1 GPU"),
            "hv_applied": hv_count, "gpu_launches": args.steps * (
                # per step: prepare (1 kernel, gather fused), cg_init x2, then T x
                # (one-pass product, fused finalize + cg_step1, cg_step2); sharded:
                # T x (product, finalize, snx_finish_hv, cg_step1, cg_step2)
                1 + 2 + T_CG * (5 if sharded else 3)),
            "clocks": clk.summary(), "roofline": roofline, "cg_kernels": cg_rate, "e2e": e2e,
            "cpu_baseline": cpu, "time_to_tolerance": solve, "trust_region_config4": tr4,
            "other_shapes": shapes, "sharded_extras": extras,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def spawn(args):
    """--gpus N > 1 without a torchrun environment: re-launch this script under
    torch.distributed.run with N ranks on 127.0.0.1; its rank 0 prints the line."""
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-solve", action="store_true")
    ap.add_argument("--skip-shapes", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
