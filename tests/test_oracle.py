"""The CPU oracle (oracle/refdyn_np.py) pinned against the reference's own
outputs (tests/golden/*.npz, made by tests/golden/make_golden.py from
/root/reference) and against the SPEC known-answer tests."""
import numpy as np
import pytest

from conftest import MODELS, golden, rel_err
from oracle import refdyn_np as R
from paper_2109_06976_b200 import models, urdf


@pytest.mark.parametrize("name", MODELS)
def test_oracle_matches_reference_outputs(name):
    g = golden(name)
    m = models.load(name)
    for alg in R.ALGORITHMS:
        out = R.evaluate_batch(m, alg, g["q"], g["qd"], g["u"])
        for nm, v in out.items():
            assert rel_err(v, g[f"{alg}.{nm}"]) < 1e-12, (name, alg, nm)


LINK = """<robot name="kat"><link name="base"/>
<link name="l"><inertial><origin xyz="1 0 0"/><mass value="1"/>
<inertia ixx="0" iyy="0" izz="0" ixy="0" ixz="0" iyz="0"/></inertial></link>
<joint name="j" type="revolute"><parent link="base"/><child link="l"/>
<axis xyz="0 0 1"/></joint></robot>"""


def test_kat_single_link_zero_gravity():
    # SPEC.md:202-203, :219, :228, :238, :246, :255
    m = urdf.parse_urdf(LINK, gravity=(0, 0, 0))
    assert R.rnea(m, [0.3], [0.0], [0.0])[0] == pytest.approx(0.0, abs=1e-15)
    assert R.rnea(m, [0.3], [0.0], [2.5])[0] == pytest.approx(2.5, abs=1e-14)
    assert np.allclose(R.crba_mass_matrix(m, [0.7]), [[1.0]], atol=1e-14)
    assert np.allclose(R.minv_direct(m, [0.7]), [[1.0]], atol=1e-14)
    assert R.forward_dynamics(m, [0.1], [0.0], [2.0])[0] == pytest.approx(2.0, abs=1e-14)
    dq, _ = R.rnea_grad(m, [0.4], [0.2], [0.1])
    assert np.allclose(dq, 0.0, atol=1e-14)
    dq, _ = R.fd_grad(m, [0.4], [0.2], [0.1])
    assert np.allclose(dq, 0.0, atol=1e-14)


@pytest.mark.parametrize("name", ["chain7", "quad12", "mixed5"])
def test_oracle_identities(name):
    # FD o ID, Minv * M_crba = I
    m = models.load(name)
    rng = np.random.default_rng(3)
    n = m.n_dof
    for _ in range(5):
        q, qd, tau = rng.uniform(-np.pi, np.pi, n), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        qdd = R.forward_dynamics(m, q, qd, tau)
        assert np.allclose(R.rnea(m, q, qd, qdd), tau, atol=1e-9)
        assert np.allclose(R.minv_direct(m, q) @ R.crba_mass_matrix(m, q), np.eye(n), atol=1e-9)


def test_oracle_gradients_vs_finite_differences():
    # central differences h = 1e-6
    m = models.load("chain7")
    rng = np.random.default_rng(4)
    n = m.n_dof
    q, qd, tau = rng.uniform(-np.pi, np.pi, n), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    dq, dqd = R.fd_grad(m, q, qd, tau)
    fq = R.finite_diff(lambda x: R.forward_dynamics(m, x, qd, tau), q, 1e-6)
    fqd = R.finite_diff(lambda x: R.forward_dynamics(m, q, x, tau), qd, 1e-6)
    assert np.max(np.abs(dq - fq)) <= 1e-5 * np.max(np.abs(fq)) + 1e-7
    assert np.max(np.abs(dqd - fqd)) <= 1e-5 * np.max(np.abs(fqd)) + 1e-7


def test_check_state_errors():
    m = models.load("chain7")
    with pytest.raises(ValueError):
        R.rnea(m, np.zeros(6), np.zeros(7), np.zeros(7))
    with pytest.raises(ValueError):
        R.rnea(m, np.full(7, np.nan), np.zeros(7), np.zeros(7))


@pytest.mark.parametrize("name", ["link1", "pendulum2", "chain7", "quad12", "humanoid30", "tree7", "mixed5"])
def test_oracle_fext_pinned_to_reference(name):
    """The oracle's f_ext path vs the reference's own outputs with seeded
    per-link external forces (tests/golden/make_golden.py, keys 'fext.*')."""
    g = golden(name)
    m = models.load(name)
    for alg in ("ID", "FD", "gradID", "gradFD"):
        r = R.evaluate_batch(m, alg, g["q"], g["qd"], g["u"], g["f_ext"])
        for nm, v in r.items():
            assert rel_err(v, g[f"fext.{alg}.{nm}"]) < 1e-12, (name, alg, nm)
