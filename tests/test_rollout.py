"""Device-resident rollouts (rollout.py): B trajectories x H semi-implicit
Euler steps on the GPU (FD or gradFD + rbd_euler_step per step, optionally
replayed from a CUDA graph) against the CPU oracle stepped the same way."""
import numpy as np
import pytest

from conftest import rel_err
from oracle import refdyn_np as R
from paper_2109_06976_b200 import models

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,B,H", [("chain7", 37, 6), ("quad12", 5, 6), ("humanoid30", 33, 2)])
@pytest.mark.parametrize("mode", ["fused", "launches", "graph"])
def test_rollout_matches_oracle(name, B, H, mode):
    """fused: one rbd_rollout launch over the horizon (2 trajectory groups,
    the last ragged, for chain7 / humanoid30; humanoid30's program uses the
    global arena); launches / graph: per-step launches, direct or replayed."""
    from paper_2109_06976_b200.rollout import Rollout
    m = models.load(name)
    n = m.n_dof
    dt = 0.01
    rng = np.random.default_rng(3)
    q0, qd0 = rng.uniform(-1, 1, (B, n)), rng.uniform(-1, 1, (B, n))
    tau = rng.uniform(-1, 1, (B, H, n))
    r = Rollout(m, B, H, dt, "f64", grad=True, graph=(mode == "graph"), fused=(mode == "fused"))
    dev = lambda x: torch.from_numpy(x).cuda()
    for _ in range(2):  # the second call replays the captured graph
        r.run(dev(q0), dev(qd0), dev(tau))
    torch.cuda.synchronize()
    q, qd, qdd, dq, dqd = (x.cpu().numpy() for x in r.trajectories())
    # oracle, stepped identically (a sample of the trajectories for the big robot)
    for b in (range(B) if n < 20 else (0, B - 1)):
        qb, qdb = q0[b].copy(), qd0[b].copy()
        for k in range(H):
            ref = R.evaluate(m, "gradFD", qb, qdb, tau[b, k])
            assert rel_err(qdd[b, k][None], ref["qdd_out"][None]) < 1e-9
            assert rel_err(dq[b, k].reshape(1, -1), ref["dq_out"][None]) < 1e-9
            assert rel_err(dqd[b, k].reshape(1, -1), ref["dqd_out"][None]) < 1e-9
            qdb = qdb + dt * ref["qdd_out"]
            qb = qb + dt * qdb
            assert rel_err(q[b, k + 1][None], qb[None]) < 1e-9
            assert rel_err(qd[b, k + 1][None], qdb[None]) < 1e-9


def test_rollout_without_gradients_and_shape_errors():
    from paper_2109_06976_b200.rollout import rollout
    m = models.load("chain7")
    n, B, H = m.n_dof, 3, 4
    q0 = torch.zeros((B, n), dtype=torch.float64, device="cuda")
    tau = torch.zeros((B, H, n), dtype=torch.float64, device="cuda")
    q, qd, qdd = rollout(m, q0, q0.clone(), tau, 0.005)
    torch.cuda.synchronize()
    assert q.shape == (B, H + 1, n) and qdd.shape == (B, H, n)
    ref = R.forward_dynamics(m, np.zeros(n), np.zeros(n), np.zeros(n))
    assert np.allclose(qdd[0, 0].cpu().numpy(), ref, rtol=1e-12, atol=1e-12)
    with pytest.raises(ValueError):
        rollout(m, q0, q0, tau[:, :, :5], 0.005)


def test_rollout_fp32():
    from paper_2109_06976_b200.rollout import Rollout
    m = models.load("chain7")
    n, B, H, dt = m.n_dof, 8, 5, 0.01
    rng = np.random.default_rng(5)
    q0, qd0 = rng.uniform(-1, 1, (B, n)).astype(np.float32), rng.uniform(-1, 1, (B, n)).astype(np.float32)
    tau = rng.uniform(-1, 1, (B, H, n)).astype(np.float32)
    r = Rollout(m, B, H, dt, "f32", grad=False, graph=True, fused=True)  # the fused FD kernel in fp32
    r.run(torch.from_numpy(q0).cuda(), torch.from_numpy(qd0).cuda(), torch.from_numpy(tau).cuda())
    torch.cuda.synchronize()
    q, qd, qdd = (x.cpu().numpy().astype(np.float64) for x in r.trajectories())
    for b in range(B):
        qb, qdb = q0[b].astype(np.float64), qd0[b].astype(np.float64)
        for k in range(H):
            ref = R.forward_dynamics(m, qb, qdb, tau[b, k].astype(np.float64))
            assert rel_err(qdd[b, k][None], ref[None]) < 1e-3  # fp32 kernels along an fp64 reference path
            qdb = qdb + dt * ref
            qb = qb + dt * qdb
        assert rel_err(q[b, H][None], qb[None]) < 1e-4
