import time, numpy as np, torch
dev = torch.device("cuda")
a = np.random.default_rng(0).standard_normal(27648)
idx = np.sort(np.random.default_rng(1).choice(50000, 2500, replace=False))
torch.cuda.synchronize()
def bench(name, fn, R=200):
    for _ in range(10): fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(R): fn()
    dt = (time.perf_counter() - t) / R * 1e6
    torch.cuda.synchronize()
    print(f"{name:40s} {dt:7.1f} us")
bench("pin_memory().to(nb)", lambda: torch.from_numpy(a).pin_memory().to(dev, non_blocking=True))
bench("pin_memory() only", lambda: torch.from_numpy(a).pin_memory())
h = torch.empty(27648, dtype=torch.float64, pin_memory=True)
hn = h.numpy()
def ring():
    np.copyto(hn, a)
    return h.to(dev, non_blocking=True)
bench("persistent pinned copyto + to(nb)", ring)
def ring2():
    np.copyto(hn, a)
    out = torch.empty(27648, dtype=torch.float64, device=dev)
    out.copy_(h, non_blocking=True)
    return out
bench("persistent pinned copyto + empty+copy_", ring2)
bench("np.copyto only", lambda: np.copyto(hn, a))
bench("torch.empty cuda", lambda: torch.empty(27648, dtype=torch.float64, device=dev))
bench("pageable .to(dev)", lambda: torch.from_numpy(a).to(dev))
bench("idx pin+to", lambda: torch.from_numpy(idx).pin_memory().to(dev, non_blocking=True))
bench("stream handle", lambda: torch.cuda.current_stream().cuda_stream)
e = torch.cuda.Event()
def ev():
    e.record(); e.query()
bench("event record+query", ev)
