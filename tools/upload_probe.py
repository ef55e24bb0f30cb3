"""Host cost of the public-API input path (e2e): numpy -> pinned -> device, per piece."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_09113_b200 import device  # noqa: E402

dev = torch.device("cuda")
torch.zeros(1, device=dev)
for n, dt in ((2500, np.int64), (27648, np.float64)):
    a = np.random.default_rng(0).random(n).astype(dt)
    R = 200
    T = {}
    for r in range(R + 20):
        t0 = time.perf_counter()
        t = torch.from_numpy(np.ascontiguousarray(a))
        t1 = time.perf_counter()
        h = t.pin_memory()
        t2 = time.perf_counter()
        d = h.to(dev, non_blocking=True)
        t3 = time.perf_counter()
        if r >= 20:
            for k, v in (("from_numpy", t1 - t0), ("pin_memory", t2 - t1), ("to(dev)", t3 - t2)):
                T[k] = T.get(k, 0) + v
    torch.cuda.synchronize()
    print(n, dt.__name__, {k: round(v / R * 1e6, 1) for k, v in T.items()})
    # persistent pinned staging + copy_
    st = torch.empty(n, dtype=torch.from_numpy(a).dtype, pin_memory=True)
    dst = torch.empty(n, dtype=st.dtype, device=dev)
    T = {}
    for r in range(R + 20):
        t0 = time.perf_counter()
        np.copyto(st.numpy(), a)
        t1 = time.perf_counter()
        dst.copy_(st, non_blocking=True)
        t2 = time.perf_counter()
        torch.cuda.current_stream().synchronize()
        if r >= 20:
            for k, v in (("memcpy to pinned", t1 - t0), ("copy_ enqueue", t2 - t1)):
                T[k] = T.get(k, 0) + v
    print("  staged:", {k: round(v / R * 1e6, 1) for k, v in T.items()})
    T = {}
    for r in range(R + 20):
        t0 = time.perf_counter()
        x = device.upload(a)
        t1 = time.perf_counter()
        if r >= 20:
            T["device.upload"] = T.get("device.upload", 0) + t1 - t0
    torch.cuda.synchronize()
    print("  device.upload:", {k: round(v / R * 1e6, 1) for k, v in T.items()})
