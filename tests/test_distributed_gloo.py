"""World-size-2 gloo tests (CPU) of the row-sharded decomposition.

The CUDA kernels cannot run here; what is tested is the host logic the
multi-GPU path relies on -- shard bounds, the split of a global sample into
shard-local indices, and that one all-reduce of per-shard partial sums (each
computed by the CPU oracle on its shard with lam = 0) plus lam * x reproduces
the full-data gradient, Hessian product, objective and accuracy.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1802_09113_b200 import distributed as sd


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, p, C, lam = 1001, 13, 5, 1e-3
        A, y = oracle.synthetic_problem(n, p, C, seed=4)
        x = 0.3 * np.random.default_rng(1).standard_normal((C - 1) * p)
        v = np.random.default_rng(2).standard_normal((C - 1) * p)
        lo, hi = sd.shard_bounds(n, world, rank)
        As, ys = A[lo:hi], y[lo:hi]
        s_g, s_h = oracle.draw_samples(0.2, 0.05, False, 7, n, 3)
        lg, lh = sd.local_indices(s_g, lo, hi), sd.local_indices(s_h, lo, hi)
        # gradient over S_g: per-shard partial with lam = 0, one all-reduce, + lam x
        g = torch.from_numpy(oracle.grad(As[lg], ys[lg], C, x, 0.0, scale=n / len(s_g)))
        sd.all_reduce_(g)
        g = g.numpy() + lam * x
        g_ref = oracle.grad(A[s_g], y[s_g], C, x, lam, scale=n / len(s_g))
        # Hessian product over S_H
        h = oracle.hess_probs(As[lh], ys[lh], C, x)
        hv = torch.from_numpy(oracle.hess_apply(As[lh], h, C, v, n / len(s_h), 0.0))
        sd.all_reduce_(hv)
        hv = hv.numpy() + lam * v
        hr = oracle.hess_probs(A[s_h], y[s_h], C, x)
        hv_ref = oracle.hess_apply(A[s_h], hr, C, v, n / len(s_h), lam)
        # objective and correct count: two scalars
        sc = torch.tensor([oracle.data_loss(As, ys, C, x),
                           float(np.sum(oracle.predict(As, ys, C, x) == ys))], dtype=torch.float64)
        sd.all_reduce_(sc)
        f = float(sc[0]) + 0.5 * lam * float(x @ x)
        # every sampled row lands on exactly one rank
        cnt = torch.tensor([len(lh), len(lg)], dtype=torch.int64)
        sd.all_reduce_(cnt)
        q.put((rank, np.linalg.norm(g - g_ref) / np.linalg.norm(g_ref),
               np.linalg.norm(hv - hv_ref) / np.linalg.norm(hv_ref),
               abs(f - oracle.loss(A, y, C, x, lam)) / abs(f),
               float(sc[1]) / n - oracle.accuracy(A, y, C, x),
               cnt.tolist(), [len(s_h), len(s_g)], sd.world_info()))
    finally:
        dist.destroy_process_group()


def test_shard_bounds_and_local_indices():
    n = 1001
    for world in (1, 2, 3, 8):
        b = [sd.shard_bounds(n, world, r) for r in range(world)]
        assert b[0][0] == 0 and b[-1][1] == n
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
        assert max(h - lo for lo, h in b) - min(h - lo for lo, h in b) <= 1
        s = oracle.draw_samples(1.0, 0.1, False, 0, n, 0)[1]
        parts = [sd.local_indices(s, lo, h) + lo for lo, h in b]
        assert np.array_equal(np.concatenate(parts), s)
    assert sd.world_info() == (1, 0)


@pytest.mark.timeout(300)
def test_two_rank_decomposition_matches_full_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, eg, ehv, ef, eacc, cnt, want, info in results:
        assert info == (2, rank)
        assert eg <= 1e-12 and ehv <= 1e-12 and ef <= 1e-13, (eg, ehv, ef)
        assert abs(eacc) < 1e-12
        assert cnt == want
