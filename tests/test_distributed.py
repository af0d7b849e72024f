"""Multi-GPU plumbing on CPU: batch sharding + optional all-gather, run with
the gloo backend at world size 2 (the GPU path uses the same code with NCCL)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2109_06976_b200 import distributed


def test_shard_bounds_cover_batch():
    for N in (0, 1, 7, 16, 1000, 1 << 20):
        for W in (1, 2, 3, 4, 8):
            b = distributed.split_even(N, W)
            assert b[0][0] == 0 and b[-1][1] == N
            assert all(b[i][1] == b[i + 1][0] for i in range(W - 1))
            sizes = [y - x for x, y in b]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        distributed.shard_bounds(10, 2, 2)


def _worker(rank, world, port, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import refdyn_np as R
    from paper_2109_06976_b200 import models
    m = models.load("pendulum2")
    rng = np.random.default_rng(0)
    N = 9
    xs = [torch.from_numpy(rng.uniform(-1, 1, (N, 2))) for _ in range(3)]

    def evaluate(parts):  # stands in for the per-GPU kernel launch
        r = R.evaluate_batch(m, "gradFD", *[p.numpy() for p in parts])
        return [torch.from_numpy(r[k]) for k in ("dq_out", "dqd_out", "qdd_out")]

    outs, bounds = distributed.run_sharded(evaluate, xs, gather_result=True)
    full = R.evaluate_batch(m, "gradFD", *[x.numpy() for x in xs])
    ok = all(np.allclose(o.numpy(), full[k]) for o, k in zip(outs, ("dq_out", "dqd_out", "qdd_out")))
    ret[rank] = (ok, bounds)
    dist.destroy_process_group()


def test_sharded_gather_gloo_world2():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    ret = mgr.dict()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, ret)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert ret[0][0] and ret[1][0]
    assert ret[0][1] == (0, 5) and ret[1][1] == (5, 9)
