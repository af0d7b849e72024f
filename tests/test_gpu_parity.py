"""GPU parity: the sm_100a kernels, called through the C ABI (device path via
torch CUDA tensors, host path via numpy + rbd_run_host), against the
reference's own outputs (golden fixtures) and the CPU oracle.

Tolerances (north star): fp64 <= 1e-9 relative, fp32 <= 1e-4 relative against
fp64 evaluation of the fp32-rounded inputs; norm-wise per knot and output
(SURVEY §8c).  Cross-tree blocks must be exact zeros."""
import numpy as np
import pytest

from conftest import MODELS, TOL, golden, rel_err
from oracle import refdyn_np as R
from paper_2109_06976_b200 import codegen, dynamics, kernels, models, program

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _dev(*xs, dt=torch.float64):
    return [torch.as_tensor(x).to("cuda", dt) for x in xs]


def _device_eval(m, alg, dt, q, qd, u):
    from paper_2109_06976_b200 import runtime
    lib = kernels.library(m)
    tdt = torch.float64 if dt == "f64" else torch.float32
    N = q.shape[0]
    xs = _dev(q, qd, u, dt=tdt)
    nin = len(codegen.INPUTS[alg])
    outs = [torch.full((N, e), float("nan"), dtype=tdt, device="cuda") for _, e in codegen.outputs(alg, m.n_dof)]
    runtime.launch(lib, alg, dt, [x.data_ptr() for x in xs[:nin]], [o.data_ptr() for o in outs], N,
                   torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return {nm: o.cpu().numpy() for (nm, _), o in zip(codegen.outputs(alg, m.n_dof), outs)}


@pytest.mark.parametrize("name", MODELS)
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_all_algorithms_match_reference(name, dt):
    g = golden(name)
    m = models.load(name)
    for alg in codegen.ALGORITHMS:
        if dt == "f64":
            q, qd, u = g["q"], g["qd"], g["u"]
            refs = {nm: g[f"{alg}.{nm}"] for nm, _ in codegen.outputs(alg, m.n_dof)}
        else:
            q, qd, u = (g[k].astype(np.float32) for k in ("q", "qd", "u"))
            refs = R.evaluate_batch(m, alg, q.astype(np.float64), qd.astype(np.float64), u.astype(np.float64))
        out = _device_eval(m, alg, dt, q, qd, u)
        for nm, v in out.items():
            assert np.all(np.isfinite(v)), (name, alg, nm)
            assert rel_err(v, refs[nm]) < TOL[dt], (name, alg, dt, nm, rel_err(v, refs[nm]))


@pytest.mark.parametrize("name", MODELS)
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_large_batch_mapping_matches_reference(name, dt):
    """Above the small-batch threshold the library launches the other kernel
    mapping (thread per knot with its register plan and parked outputs):
    golden knots tiled to N = threshold + 37 (ragged last CTA), every knot
    checked."""
    g = golden(name)
    m = models.load(name)
    N = int(codegen.tuning(m, "gradFD", dt)["ws_max_n"]) + 37
    reps = -(-N // g["q"].shape[0])
    tile = lambda x: np.tile(x, (reps, 1))[:N]
    for alg in codegen.ALGORITHMS:
        if dt == "f64":
            q, qd, u = (tile(g[k]) for k in ("q", "qd", "u"))
            refs = {nm: tile(g[f"{alg}.{nm}"]) for nm, _ in codegen.outputs(alg, m.n_dof)}
        else:
            q32, qd32, u32 = (g[k].astype(np.float32) for k in ("q", "qd", "u"))
            r = R.evaluate_batch(m, alg, q32.astype(np.float64), qd32.astype(np.float64), u32.astype(np.float64))
            q, qd, u = tile(q32), tile(qd32), tile(u32)
            refs = {nm: tile(v) for nm, v in r.items()}
        out = _device_eval(m, alg, dt, q, qd, u)
        for nm, v in out.items():
            assert np.all(np.isfinite(v)), (name, alg, nm)
            assert rel_err(v, refs[nm]) < TOL[dt], (name, alg, dt, nm, rel_err(v, refs[nm]))


@pytest.mark.parametrize("name", MODELS)
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_mid_batch_mapping(name, dt):
    """Mid-size batches (below the large-batch threshold, several CTAs of the
    warp-specialised kernel, ragged last group): golden knots tiled to
    N = 1000, gradFD."""
    g = golden(name)
    m = models.load(name)
    N = 1000
    reps = -(-N // g["q"].shape[0])
    tile = lambda x: np.tile(x, (reps, 1))[:N]
    if dt == "f64":
        q, qd, u = (tile(g[k]) for k in ("q", "qd", "u"))
        refs = {nm: tile(g[f"gradFD.{nm}"]) for nm, _ in codegen.outputs("gradFD", m.n_dof)}
    else:
        q32, qd32, u32 = (g[k].astype(np.float32) for k in ("q", "qd", "u"))
        r = R.evaluate_batch(m, "gradFD", q32.astype(np.float64), qd32.astype(np.float64), u32.astype(np.float64))
        q, qd, u = tile(q32), tile(qd32), tile(u32)
        refs = {nm: tile(v) for nm, v in r.items()}
    out = _device_eval(m, "gradFD", dt, q, qd, u)
    for nm, v in out.items():
        assert rel_err(v, refs[nm]) < TOL[dt], (name, dt, nm)


@pytest.mark.parametrize("name", ["quad12", "humanoid30"])
def test_cross_tree_blocks_exact_zero(name):
    g = golden(name)
    m = models.load(name)
    root = [m.root_of(i) for i in range(m.n_dof)]
    mask = np.array([[root[i] != root[j] for j in range(m.n_dof)] for i in range(m.n_dof)])
    for alg in ("Minv", "gradID", "gradFD"):
        out = _device_eval(m, alg, "f64", g["q"], g["qd"], g["u"])
        for nm, v in out.items():
            if v.shape[1] == m.n_dof ** 2:
                assert np.all(v.reshape(-1, m.n_dof, m.n_dof)[:, mask] == 0.0)


@pytest.mark.parametrize("N", [0, 1, 63, 64, 65, 127, 1000])
def test_ragged_batch_sizes(N):
    m = models.load("chain7")
    rng = np.random.default_rng(N)
    n = m.n_dof
    q, qd, u = rng.uniform(-np.pi, np.pi, (N, n)), rng.uniform(-1, 1, (N, n)), rng.uniform(-1, 1, (N, n))
    out = _device_eval(m, "gradFD", "f64", q, qd, u)
    if N == 0:
        assert all(v.shape[0] == 0 for v in out.values())
        return
    ref = R.evaluate_batch(m, "gradFD", q, qd, u)
    for nm in ref:
        assert rel_err(out[nm], ref[nm]) < 1e-9


def test_drop_in_api_host_and_device():
    m = models.load("quad12")
    g = golden("quad12")
    # single knot (n,), numpy -> host-buffer path, reference return shapes
    k = 3
    tau = dynamics.rnea(m, g["q"][k], g["qd"][k], g["u"][k])
    assert tau.shape == (12,) and rel_err(tau[None], g["ID.tau_out"][k:k + 1]) < 1e-9
    Mi = dynamics.minv_direct(m, g["q"][k])
    assert Mi.shape == (12, 12) and rel_err(Mi.reshape(1, -1), g["Minv.minv_out"][k:k + 1]) < 1e-9
    gr = dynamics.fd_grad(m, g["q"], g["qd"], g["u"])
    assert gr.dq.shape == (16, 12, 12)
    assert rel_err(gr.dq, g["gradFD.dq_out"]) < 1e-9 and rel_err(gr.dqd, g["gradFD.dqd_out"]) < 1e-9
    # device tensors stay on the device
    gd = dynamics.rnea_grad(m, *_dev(g["q"], g["qd"], g["u"]))
    assert gd.dq.is_cuda
    assert rel_err(gd.dq.cpu().numpy(), g["gradID.dq_out"]) < 1e-9
    qdd = dynamics.forward_dynamics(m, *_dev(g["q"], g["qd"], g["u"], dt=torch.float32))
    assert qdd.dtype == torch.float32
    c = dynamics.bias_force(m, g["q"], g["qd"])
    assert np.allclose(dynamics.forward_dynamics(m, g["q"], g["qd"], c), 0.0, atol=1e-10)


def test_operator_api_build_interpret():
    m = models.load("chain7")
    g = golden("chain7")
    prog, sched, layout = program.build(m, "gradFD")
    assert set(prog.input_map) == {"q", "qd", "tau"}
    assert list(prog.output_map) == ["dq_out", "dqd_out", "qdd_out"]
    out = program.interpret(prog, {"q": g["q"][0], "qd": g["qd"][0], "tau": g["u"][0]})
    assert out["dq_out"].shape == (49,)
    assert rel_err(out["dq_out"][None], g["gradFD.dq_out"][:1]) < 1e-9
    with pytest.raises(program.InterpreterError):
        program.interpret(prog, {"q": g["q"][0], "qd": g["qd"][0]})
    with pytest.raises(program.InterpreterError):
        program.interpret(prog, {"q": g["q"][0][:5], "qd": g["qd"][0], "tau": g["u"][0]})


def test_errors_like_reference():
    m = models.load("chain7")
    with pytest.raises(ValueError):
        dynamics.rnea(m, np.zeros(6), np.zeros(7), np.zeros(7))
    with pytest.raises(ValueError):
        dynamics.rnea(m, np.full(7, np.inf), np.zeros(7), np.zeros(7))
    with pytest.raises(ValueError):  # f_ext must be (n, 6) for one knot
        dynamics.rnea(m, np.zeros(7), np.zeros(7), np.zeros(7), f_ext=np.zeros((7, 5)))
    with pytest.raises(ValueError):
        dynamics.rnea(m, np.zeros(7), np.zeros(7), np.zeros(7), f_ext=np.full((7, 6), np.nan))


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_nonfinite_inputs_rejected_on_device(dt):
    """Large host batches are checked on the device, chunk by chunk: one NaN
    deep in a later chunk raises ValueError (refdyn._check_state), and the
    session's flag is re-armed for the next call."""
    m = models.load("chain7")
    ndt = np.float64 if dt == "f64" else np.float32
    rng = np.random.default_rng(4)
    N = 300_000  # several pipeline chunks
    q, qd, tau = (rng.uniform(-1, 1, (N, 7)).astype(ndt) for _ in range(3))
    bad = qd.copy()
    bad[N - 17, 3] = np.nan
    with pytest.raises(ValueError):
        dynamics.forward_dynamics(m, q, bad, tau)
    bad = tau.copy()
    bad[123_456, 0] = np.inf
    with pytest.raises(ValueError):
        dynamics.fd_grad(m, q, qd, bad)
    qdd = dynamics.forward_dynamics(m, q[:64], qd[:64], tau[:64])
    ref = R.evaluate_batch(m, "FD", *(x[:64].astype(np.float64) for x in (q, qd, tau)))["qdd_out"]
    assert rel_err(qdd, ref) < TOL[dt]
    qdd = dynamics.forward_dynamics(m, q, qd, tau)  # flag re-armed after the failures
    assert np.all(np.isfinite(qdd))


@pytest.mark.parametrize("name", MODELS)
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_fext_matches_reference(name, dt):
    """The f_ext entries (refdyn's f_ext argument) against the reference's
    own outputs with seeded external forces, on both kernel mappings (golden
    knots, and tiled past the small-batch threshold), device and host paths."""
    g = golden(name)
    m = models.load(name)
    n = m.n_dof
    big = int(codegen.tuning(m, "gradFD", dt)["ws_max_n"]) + 37
    for N in (g["q"].shape[0], big):
        reps = -(-N // g["q"].shape[0])
        tile = lambda x: np.tile(x, (reps,) + (1,) * (x.ndim - 1))[:N]
        q, qd, u, fx = (tile(g[k]) for k in ("q", "qd", "u", "f_ext"))
        tdt = torch.float64 if dt == "f64" else torch.float32
        for alg in codegen.FEXT_ALGORITHMS:
            if dt == "f64":
                refs = {nm: tile(g[f"fext.{alg}.{nm}"]) for nm, _ in codegen.outputs(alg, n)}
            else:
                r32 = [g[k].astype(np.float32).astype(np.float64) for k in ("q", "qd", "u", "f_ext")]
                refs = {k: tile(v) for k, v in R.evaluate_batch(m, alg, *r32).items()}
            xs = _dev(q, qd, u, fx, dt=tdt)
            fn = {"ID": dynamics.rnea, "FD": dynamics.forward_dynamics, "gradID": dynamics.rnea_grad,
                  "gradFD": dynamics.fd_grad}[alg]
            got = fn(m, *xs[:3], f_ext=xs[3])
            torch.cuda.synchronize()
            vals = [got] if alg in ("ID", "FD") else ([got.dq, got.dqd] + ([got.qdd] if alg == "gradFD" else []))
            for (nm, _), v in zip(codegen.outputs(alg, n), vals):
                v = v.cpu().numpy().reshape(N, -1)
                assert rel_err(v, refs[nm]) < TOL[dt], (name, alg, dt, N, nm, rel_err(v, refs[nm]))
        if dt == "f32":
            continue
        # host path (numpy in, numpy out) through rbd_run_host_fext: zero-copy
        # at the golden N, the chunked H2D / kernel / D2H pipeline at the big N
        got = dynamics.fd_grad(m, q, qd, u, f_ext=fx)
        assert rel_err(got.dq.reshape(N, -1), tile(g["fext.gradFD.dq_out"])) < 1e-9
        assert rel_err(got.qdd.reshape(N, -1), tile(g["fext.gradFD.qdd_out"])) < 1e-9
        if N == big:
            continue
        one = dynamics.rnea(m, q[0], qd[0], u[0], f_ext=fx[0])
        assert rel_err(one[None], g["fext.ID.tau_out"][:1]) < 1e-9


FULL_SIZE = [("chain7", "f64", 1 << 20), ("chain7", "f32", 1 << 20),
             ("quad12", "f64", 1 << 20), ("quad12", "f32", 1 << 20),
             ("humanoid30", "f64", 1 << 18), ("humanoid30", "f32", 1 << 18),
             ("humanoid30", "f64", 1 << 20), ("humanoid30", "f32", 1 << 20)]


@pytest.mark.parametrize("name,dt,N", FULL_SIZE)
def test_full_size_properties(name, dt, N):
    """Every benchmarked large-batch config (BASELINE configs[4] sizes): 64
    sampled knots of gradFD vs the oracle at the north-star tolerance, plus
    size-independent identities over the whole batch on the device:
    ID(q, qd, FD(q, qd, tau)) = tau, FD qdd = gradFD qdd, Minv symmetric,
    cross-tree blocks of dFD exactly 0.

    The identity tolerance is 1e-9 (fp64) / 1e-4 (fp32) relative to the
    magnitude of the terms the RNEA sums, max|tau| + max|c(q, qd)|: tau is
    U(-1, 1) while the bias c reaches tens of N m, so a backward-stable fp32
    round trip is accurate to eps * |c|, not to eps * |tau|."""
    m = models.load(name)
    n = m.n_dof
    tdt = torch.float64 if dt == "f64" else torch.float32
    gen = torch.Generator(device="cuda").manual_seed(5)
    q = (torch.rand((N, n), generator=gen, device="cuda", dtype=torch.float64) * 2 - 1) * np.pi
    qd = torch.rand((N, n), generator=gen, device="cuda", dtype=torch.float64) * 2 - 1
    tau = torch.rand((N, n), generator=gen, device="cuda", dtype=torch.float64) * 2 - 1
    q, qd, tau = q.to(tdt), qd.to(tdt), tau.to(tdt)
    g = dynamics.fd_grad(m, q, qd, tau)
    torch.cuda.synchronize()
    idx = torch.randint(0, N, (64,), generator=gen, device="cuda").cpu().numpy()
    idx[0], idx[-1] = 0, N - 1  # first and last CTA / chunk
    qs, qds, taus = (x[idx].double().cpu().numpy() for x in (q, qd, tau))
    ref = R.evaluate_batch(m, "gradFD", qs, qds, taus)
    for nm, v in (("dq_out", g.dq), ("dqd_out", g.dqd), ("qdd_out", g.qdd)):
        assert rel_err(v[idx].reshape(len(idx), -1).double().cpu().numpy(), ref[nm]) < TOL[dt], (name, dt, N, nm)
    blocks = np.zeros((n, n), dtype=bool)
    for t in m.roots():
        sub = m.subtree(t)
        blocks[np.ix_(sub, sub)] = True
    if not blocks.all():
        off = torch.from_numpy(~blocks).cuda()
        assert float(g.dq[:, off].abs().max()) == 0.0 and float(g.dqd[:, off].abs().max()) == 0.0
    gqdd = g.qdd
    del g
    qdd = dynamics.forward_dynamics(m, q, qd, tau)
    assert float(((gqdd - qdd).abs().amax(dim=1) / qdd.abs().amax(dim=1).clamp_min(1e-30)).max()) < TOL[dt]
    del gqdd
    tau2 = dynamics.rnea(m, q, qd, qdd)
    c = dynamics.bias_force(m, q, qd)
    scale = tau.abs().amax(dim=1) + c.abs().amax(dim=1)
    assert float(((tau2 - tau).abs().amax(dim=1) / scale).max()) < TOL[dt], (name, dt, N)
    del tau2, c, qdd
    Mi = dynamics.minv_direct(m, q)
    assert float((Mi - Mi.transpose(1, 2)).abs().max()) <= (1e-12 if dt == "f64" else 1e-5) * float(Mi.abs().max())


@pytest.mark.parametrize("pinned", [False, True])
def test_host_path_zero_copy_and_chunked(pinned):
    """rbd_run_host: small batches go zero-copy (pinned caller buffers in
    place, pageable ones through the session's pinned stage); large batches
    take the chunked H2D/kernel/D2H pipeline."""
    from paper_2109_06976_b200 import runtime
    for name, N in (("chain7", 100), ("quad12", 20000)):
        m = models.load(name)
        lib = kernels.library(m)
        rng = np.random.default_rng(N)
        n = m.n_dof
        xs = [rng.uniform(-np.pi, np.pi, (N, n)), rng.uniform(-1, 1, (N, n)), rng.uniform(-1, 1, (N, n))]
        outs = [np.full((N, e), np.nan) for _, e in codegen.outputs("gradFD", n)]
        keep = []
        if pinned:
            tx = [torch.from_numpy(x).pin_memory() for x in xs]
            to = [torch.from_numpy(o).pin_memory() for o in outs]
            keep = tx + to
            xs, outs = [t.numpy() for t in tx], [t.numpy() for t in to]
        runtime.run_host(lib, "gradFD", "f64", xs, outs, N)
        idx = rng.choice(N, size=min(N, 20), replace=False)
        ref = R.evaluate_batch(m, "gradFD", xs[0][idx], xs[1][idx], xs[2][idx])
        for (nm, _), o in zip(codegen.outputs("gradFD", n), outs):
            assert rel_err(o[idx], ref[nm]) < 1e-9, (name, N, nm)
        del keep


@pytest.mark.parametrize("name", ["chain7", "quad12"])
def test_large_joint_angles(name):
    """The thread-per-knot fp64 kernels evaluate the joints' sin/cos side by
    side (rbd_sincos_batch: two-part pi/2 reduction up to |q| = 2^20, the
    libdevice fallback beyond): angles across both ranges, and exact
    multiples of pi/2, match the oracle (numpy sin/cos) at 1e-9."""
    m = models.load(name)
    n = m.n_dof
    N = 8448  # above ws_max_n: the thread-per-knot kernel
    rng = np.random.default_rng(11)
    mag = 10.0 ** rng.uniform(-3, 7.5, (N, n))  # 1e-3 .. 3e7 rad, both sides of 2^20
    q = mag * rng.choice([-1.0, 1.0], (N, n))
    q[:64] = (np.pi / 2) * rng.integers(-2000, 2000, (64, n))  # reduction edge cases
    qd, tau = rng.uniform(-1, 1, (N, n)), rng.uniform(-1, 1, (N, n))
    got = _device_eval(m, "gradFD", "f64", q, qd, tau)
    idx = np.concatenate([np.arange(64), rng.integers(64, N, 64)])
    ref = R.evaluate_batch(m, "gradFD", q[idx], qd[idx], tau[idx])
    for nm in ("dq_out", "dqd_out", "qdd_out"):
        assert rel_err(got[nm][idx].reshape(len(idx), -1), ref[nm]) < TOL["f64"], (name, nm)
