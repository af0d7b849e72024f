"""Reentrancy of the C ABI (rbd_b200.h: any host thread, any stream) and the
multi-device host path, on the GPU against the oracle.

Four host threads run at once, each on its own CUDA stream:
humanoid30 gradFD at N = 256 (warp-specialised kernel, global arena shared
by every stream -> event chain), humanoid30 gradFD at N = 2^16 (the split
pipeline's per-stream scratch), and chain7 / humanoid30 numpy host calls
(per-thread sessions; the humanoid30 one is multi-chunk through the split
pipeline, the pattern the advisor's race needed)."""
import threading

import numpy as np
import pytest

from conftest import TOL, rel_err
from oracle import refdyn_np as R
from paper_2109_06976_b200 import codegen, dynamics, models, runtime

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _states(n, N, seed):
    rng = np.random.default_rng(seed)
    return (rng.uniform(-np.pi, np.pi, (N, n)), rng.uniform(-1, 1, (N, n)), rng.uniform(-1, 1, (N, n)))


def _check(m, xs, got, sample=16, seed=0):
    N = xs[0].shape[0]
    idx = np.random.default_rng(seed).choice(N, size=min(N, sample), replace=False)
    ref = R.evaluate_batch(m, "gradFD", *(x[idx] for x in xs))
    for nm, v in zip(("dq_out", "dqd_out", "qdd_out"), got):
        assert rel_err(np.asarray(v).reshape(N, -1)[idx], ref[nm]) < TOL["f64"], nm


def test_four_threads_own_streams():
    h30, c7 = models.load("humanoid30"), models.load("chain7")
    jobs = []  # (model, host states, kind)
    jobs.append((h30, _states(h30.n_dof, 256, 1), "device"))
    jobs.append((h30, _states(h30.n_dof, 1 << 16, 2), "device"))
    jobs.append((c7, _states(c7.n_dof, 50000, 3), "host"))
    jobs.append((h30, _states(h30.n_dof, 20000, 4), "host"))
    results, errors = [None] * len(jobs), []
    start = threading.Barrier(len(jobs))

    def work(k):
        try:
            m, xs, kind = jobs[k]
            torch.cuda.set_device(0)
            if kind == "device":
                st = torch.cuda.Stream()
                with torch.cuda.stream(st):
                    dx = [torch.from_numpy(x).cuda() for x in xs]
                    st.synchronize()
                    start.wait()
                    outs = []
                    for _ in range(3):  # repeated launches interleave with the other threads
                        g = dynamics.fd_grad(m, *dx)
                        outs.append(g)
                    st.synchronize()
                    results[k] = [(o.dq.cpu().numpy(), o.dqd.cpu().numpy(), o.qdd.cpu().numpy()) for o in outs]
            else:
                start.wait()
                results[k] = []
                for _ in range(3):
                    g = dynamics.fd_grad(m, *xs)
                    results[k].append((g.dq, g.dqd, g.qdd))
        except Exception as e:  # pragma: no cover - reported below
            errors.append((k, repr(e)))

    th = [threading.Thread(target=work, args=(k,)) for k in range(len(jobs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for (m, xs, _), res in zip(jobs, results):
        for got in res:
            _check(m, xs, got)


def test_multi_device_host_path():
    """dynamics.*(..., devices=[...]) -> rbd_run_host_multi: contiguous slices,
    one session + host thread each.  On a one-GPU box the list names device 0
    three times (three sessions, three concurrent pipelines); every knot must
    come back in place."""
    for name, N in (("chain7", 100003), ("humanoid30", 9001)):
        m = models.load(name)
        xs = _states(m.n_dof, N, 7)
        g = dynamics.fd_grad(m, *xs, devices=[0, 0, 0])
        _check(m, xs, (g.dq, g.dqd, g.qdd), sample=32)
        # the slice boundaries are exactly where rbd_shard puts them
        for b, ln in runtime.shard_ranges(N, 3):
            k = b + ln - 1
            ref = R.evaluate_batch(m, "gradFD", *(x[k:k + 1] for x in xs))
            assert rel_err(g.qdd.reshape(N, -1)[k:k + 1], ref["qdd_out"]) < TOL["f64"]


def _rank_worker(rank, world, port, ret):
    import os
    import sys
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import refdyn_np as R
    from paper_2109_06976_b200 import distributed, dynamics, models
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)  # both ranks share the one GPU of the box
    m = models.load("chain7")
    rng = np.random.default_rng(0)
    N = 1001
    xs = [torch.from_numpy(rng.uniform(-1, 1, (N, m.n_dof))) for _ in range(3)]
    dev = [x.cuda() for x in xs]
    outs, bounds = distributed.evaluate_sharded(dynamics.fd_grad, m, *dev)
    torch.cuda.synchronize()
    outs = [o.cpu().reshape(o.shape[0], -1) for o in outs]
    full = [distributed.gather(o, N) for o in outs]  # gloo: host tensors
    ref = R.evaluate_batch(m, "gradFD", *[x.numpy() for x in xs])
    ok = all(float(np.max(np.abs(f.numpy() - ref[k]))) <= 1e-9 * float(np.max(np.abs(ref[k])))
             for f, k in zip(full, ("dq_out", "dqd_out", "qdd_out")))
    ret[rank] = (ok, bounds)
    dist.destroy_process_group()


def test_two_ranks_shard_real_kernels():
    """distributed.evaluate_sharded with the generated kernels: world size 2
    (gloo, both ranks on cuda:0), each rank its slice, all-gathered back."""
    import os
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    ret = mgr.dict()
    port = 29700 + os.getpid() % 1000
    procs = [ctx.Process(target=_rank_worker, args=(r, 2, port, ret)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs)
    assert ret[0][0] and ret[1][0]
    assert ret[0][1] == (0, 501) and ret[1][1] == (501, 1001)
