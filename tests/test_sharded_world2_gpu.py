"""The row-sharded solver at world size 2: two processes, each
holding half of the rows, running newton_solve_sharded with real all-reduces
of the partial gradients / Hessian products / objective scalars (gloo over
CUDA tensors -- this image's test boxes have one GPU, so both ranks share
cuda:0; gloo stages the sums through the host, so no rank's kernel waits on
the other's).  The trace and the final iterate must match the single-process
CPU oracle (the reference's arithmetic), including a Hessian sample so small
that one rank holds none of its rows (its partial is zero, the all-reduce
still runs)."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
from conftest import rel_err

pytestmark = pytest.mark.gpu

CASES = {
    # name: (n, p, C, variant, f_g, f_h, iters, seed)
    "subsampled20": (3000, 40, 7, "subsampled-20", None, None, 4, 5),
    "tiny_hessian_sample": (600, 24, 4, "subsampled-100", 1.0, 0.004, 4, 3),
    # fp64 with many classes (library DGEMMs + row kernels on each shard)
    "wide_classes_c40": (1600, 48, 40, "subsampled-20", None, None, 3, 9),
}


def _worker(rank, world, port, case, out_dir):
    import torch.distributed as dist

    import paper_1802_09113_b200 as snx
    from paper_1802_09113_b200 import distributed as sd

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, p, C, variant, f_g, f_h, iters, seed = CASES[case]
    A, y = oracle.synthetic_problem(n, p, C, seed=seed)
    sp = sd.ShardedProblem.from_global(A, y, C, 1e-3)
    cfg = snx.make_variant(variant, snx.NewtonConfig(max_outer_iters=iters))
    if f_h is not None:
        cfg = snx.NewtonConfig(max_outer_iters=iters,
                               samples=snx.SampleConfig(gradient_fraction=f_g,
                                                        hessian_fraction=f_h))
    local_h = [len(sd.local_indices(sd.ShardedOracle(sp, cfg.samples, k).s_h, sp.row0,
                                    sp.row1)) for k in range(iters)]
    tr = sd.newton_solve_sharded(sp, cfg)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), x=tr.x_final,
             recs=np.array([[r.iteration, r.objective, r.train_acc, r.step_size, r.cg_iters]
                            for r in tr.records]), reason=np.array(tr.reason),
             local_h=np.array(local_h))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case", sorted(CASES))
def test_world2_sharded_newton_matches_oracle(case):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n, p, C, variant, f_g, f_h, iters, seed = CASES[case]
    with tempfile.TemporaryDirectory() as td:
        mp.start_processes(_worker, args=(2, _free_port(), case, td), nprocs=2, join=True,
                           start_method="spawn")
        got = [dict(np.load(os.path.join(td, f"rank{r}.npz"))) for r in range(2)]
    A, y = oracle.synthetic_problem(n, p, C, seed=seed)
    ref = oracle.newton_solve(A, y, C, 1e-3, variant, max_outer_iters=iters,
                              gradient_fraction=f_g, hessian_fraction=f_h)
    # every rank returns the same trace
    assert np.array_equal(got[0]["x"], got[1]["x"])
    assert np.array_equal(got[0]["recs"], got[1]["recs"])
    recs = got[0]["recs"]
    assert str(got[0]["reason"]) == ref["reason"]
    assert len(recs) == len(ref["records"])
    for (k, f, acc, step, it), (rk, rf, racc, _, ralpha, rit) in zip(recs, ref["records"]):
        assert int(k) == rk and int(it) == rit and step == ralpha
        assert abs(f - rf) <= 1e-10 * abs(rf)
        assert abs(acc - racc) <= 1e-12
    assert rel_err(got[0]["x"], ref["x"]) <= 1e-9
    if case == "tiny_hessian_sample":  # some iteration leaves one rank without sample rows
        lh = np.stack([got[0]["local_h"], got[1]["local_h"]])
        assert (lh == 0).any(), lh
