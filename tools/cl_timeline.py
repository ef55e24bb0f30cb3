"""Per-CTA, per-block timeline of the one-pass cluster kernel (debug build).

    python -c "from paper_1802_09113_b200 import _build; _build.build_timeline('tools/libsnx_cltl.so', ['-DSNX_CL_TIMELINE'])"
    SNX_LIB=tools/libsnx_cltl.so python tools/cl_timeline.py [cifar|mnist|covertype] [b2b|sync|prep|cg]

Events per block, compute thread 0: 0 loop top, 1 next block's V done,
2 U(b) ready (waited), 3 X^T U(b) done; exchange-warp lane 0: 6 warp partials
ready, 7 sent to the peers, 8 peers' partials in, 9 U rows written.  Kernel
row (-1): 0 entry, 6 shared memory zeroed, 7 cluster barrier, 8 PDL wait
done, 9 weight fragments in registers, 1 weights loaded, 2 first V done, 3 loop
end, 4 partial written, 5 exit."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_09113_b200 as snx  # noqa: E402
from paper_1802_09113_b200 import _lib  # noqa: E402

SHAPES = {"cifar": (50000, 3072, 10), "mnist": (60000, 784, 10), "covertype": (581012, 54, 7)}
name = sys.argv[1] if len(sys.argv) > 1 else "cifar"
n, p, C = SHAPES[name]
gen = np.random.default_rng(0)
A = gen.standard_normal((n, p))
A /= np.sqrt((A ** 2).sum(axis=0))
y = gen.integers(0, C, size=n)
ds = snx.DeviceDataset.from_numpy(A, y, C)
x = torch.from_numpy(0.01 * np.random.default_rng(7).standard_normal((C - 1) * p)).cuda()
orc = snx.SubsampledOracle(snx.SoftmaxProblem(ds, 1e-3), snx.SampleConfig(1.0, 0.05), 0)
g, _ = orc.gradient_device(x)
op = orc.hessian_operator(x)
out = torch.empty_like(g)
mode = sys.argv[2] if len(sys.argv) > 2 else "b2b"
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if mode == "prep":
    run = lambda: orc.hessian_operator(x)  # noqa: E731
elif mode == "grad":  # the full-data gradient pass
    run = lambda: orc.gradient_device(x)  # noqa: E731
elif mode == "cg":  # the products of a captured CG solve (the stamps: its last product)
    from paper_1802_09113_b200 import cg as cgmod
    run = lambda: cgmod.cg_graph_for(op, 10, 1e-12).run(g)  # noqa: E731
else:
    run = lambda: op.apply_into(g, out)  # noqa: E731
for _ in range(5):
    run()
torch.cuda.synchronize()
e0.record(st)
for _ in range(20):
    run()
e1.record(st)
torch.cuda.synchronize()
print(f"20 back-to-back {'prepares' if mode == 'prep' else 'products'}: "
      f"{e0.elapsed_time(e1) / 20 * 1e3:.1f} us each (events)")
if mode == "cg":
    torch.cuda.synchronize()
if mode == "sync":  # the stamps below: one product on an idle GPU
    op.apply_into(g, out)
    torch.cuda.synchronize()
NB = 26
buf = (ctypes.c_ulonglong * (160 * NB * 10))()
_lib.load().snx_debug_cl_timeline(buf)
t = np.frombuffer(buf, dtype=np.uint64).reshape(160, NB, 10).astype(np.int64)
used = [c for c in range(160) if t[c, 0, 0] != 0]
if not used:
    sys.exit(f'{name}: no stamps (kernel not used for this shape?)')
t0 = min(t[c, 0, 0] for c in used)
rel = lambda v: (v - t0) / 1e3 if v else float("nan")  # noqa: E731
print(f"{name}: {len(used)} CTAs; kernel rows: entry / smem zeroed / cluster sync / pdl wait / "
      "Q frags / Q loaded / first V / loop end / partial out / exit (us)")
for c in used[:6] + used[-2:]:
    print(f"cta {c:3d}: " + " ".join(f"{rel(t[c, 0, e]):7.2f}" for e in (0, 6, 7, 8, 9, 1, 2, 3, 4, 5)))
print("per block (cta 0): compute top / V(b+1) done / U(b) ready / XtU done | xchg red in / sent / peers in / U out")
for b in range(NB - 1):
    if t[used[0], b + 1, 0] == 0 or t[used[0], b + 1, 0] < t0:
        break
    r = t[used[0], b + 1]
    print(f"b{b:2d}: " + " ".join(f"{rel(r[e]):7.2f}" for e in range(4)) + " | " +
          " ".join(f"{rel(r[e]):7.2f}" for e in (6, 7, 8, 9)))
# medians of the phase durations over CTAs and blocks
d = {k: [] for k in ("vphase", "u_wait", "xtu", "xchg_send", "xchg_peers", "xchg_rows")}
for c in used:
    for b in range(NB - 1):
        r = t[c, b + 1]
        if r[0] == 0 or r[3] == 0 or r[0] < t0:
            continue
        d["vphase"].append(r[1] - r[0])
        d["u_wait"].append(r[2] - r[1])
        d["xtu"].append(r[3] - r[2])
        if r[9] > 0:
            d["xchg_send"].append(r[7] - r[6])
            d["xchg_peers"].append(r[8] - r[7])
            d["xchg_rows"].append(r[9] - r[8])
print("median phase us: " + ", ".join(f"{k} {np.median(v) / 1e3:.3f}" for k, v in d.items() if v))
if mode in ("b2b", "sync"):  # the last product's finalize (same clock)
    cr = (ctypes.c_ulonglong * (256 * 6))()
    _lib.load().snx_debug_cgr_timeline(cr)
    cr = np.frombuffer(cr, dtype=np.uint64).reshape(256, 6).astype(np.int64)
    ok = cr[:, 0] >= t0
    if ok.any():
        ext = np.array([t[c, 0, 5] for c in used])
        print(f"product exit med {rel(np.median(ext)):7.2f} max {rel(ext.max()):7.2f}; finalize "
              f"entry {rel(cr[ok, 0].min()):7.2f} dependency met {rel(np.median(cr[ok, 1])):7.2f}"
              f" exit med {rel(np.median(cr[ok, 2])):7.2f} max {rel(cr[ok, 2].max()):7.2f}")
