"""How much does clock sampling during the timed region perturb a bench step?"""
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1802_09113_b200 as snx  # noqa: E402
from paper_1802_09113_b200 import cg as cgmod, softmax  # noqa: E402

N, P, C = 50000, 3072, 10
A, y = oracle.synthetic_problem(N, P, C, seed=0)
ds = snx.DeviceDataset.from_numpy(A, y, C)
x = torch.from_numpy(0.01 * np.random.default_rng(7).standard_normal((C - 1) * P)).cuda()
g, _ = softmax.gradient_parts(ds, x, 1.0, 1e-3)
views = [ds.take(snx.draw_samples(snx.SampleConfig(1.0, 0.05), N, k)[1]) for k in range(40)]
st = torch.cuda.current_stream()


def step(k):
    o = softmax.HessianOperator(views[k % 40], x, 1e-3, scale=N / 2500)
    cgmod.cg_graph_for(o, 10, 1e-4).run(g)


def timed(reps=200):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for k in range(reps):
        step(k)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for k in range(5):
    step(k)
print("none                 %.1f us" % timed())

for lms in (50, 200, 1000):
    p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,clocks.max.sm",
                          "--format=csv,noheader,nounits", "-lms", str(lms)],
                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    time.sleep(0.5)
    t = timed()
    p.terminate()
    out, _ = p.communicate()
    print("nvidia-smi -lms %-4d  %.1f us  (%d samples)" % (lms, t, len(out.splitlines())))

import pynvml  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
for period, reasons in ((0.05, False), (0.05, True), (0.2, True)):
    stop = threading.Event()
    got = []

    def loop():
        while not stop.is_set():
            c = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h) if reasons else 0
            got.append((c, r))
            stop.wait(period)

    th = threading.Thread(target=loop, daemon=True)
    th.start()
    time.sleep(0.2)
    t0 = time.perf_counter()
    c0 = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    q = time.perf_counter() - t0
    t = timed()
    stop.set()
    th.join()
    print("nvml %.2fs reasons=%d  %.1f us  (%d samples, one query %.0f us, %s)"
          % (period, reasons, t, len(got), q * 1e6, got[-1]))
