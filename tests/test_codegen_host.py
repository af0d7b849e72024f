"""Generator correctness on CPU: the emitted one-knot programs, compiled for
the host by the test-only harness (tests/support/hostbuild.py), match the
reference's outputs (golden fixtures) for every robot x algorithm x dtype.
The same source compiled for sm_100a is checked on the GPU by test_gpu_parity.py."""
import numpy as np
import pytest

from conftest import MODELS, TOL, golden, rel_err
from oracle import refdyn_np as R
from paper_2109_06976_b200 import codegen, models
from support import hostbuild


@pytest.mark.parametrize("name", MODELS)
def test_generated_program_matches_reference(name):
    g = golden(name)
    m = models.load(name)
    lib = hostbuild.host_library(m)
    for alg in codegen.ALGORITHMS:
        out = hostbuild.host_eval(lib, m, alg, "f64", g["q"], g["qd"], g["u"])
        for nm, v in out.items():
            assert rel_err(v, g[f"{alg}.{nm}"]) < TOL["f64"], (name, alg, nm)
        q32, qd32, u32 = (g[k].astype(np.float32) for k in ("q", "qd", "u"))
        ref = R.evaluate_batch(m, alg, q32.astype(np.float64), qd32.astype(np.float64), u32.astype(np.float64))
        out = hostbuild.host_eval(lib, m, alg, "f32", q32, qd32, u32)
        for nm, v in out.items():
            assert rel_err(v, ref[nm]) < TOL["f32"], (name, alg, nm, "f32")


@pytest.mark.parametrize("name", ["quad12", "humanoid30"])
def test_cross_tree_blocks_are_exact_zeros(name):
    # cross-limb gradient blocks are exactly 0
    g = golden(name)
    m = models.load(name)
    lib = hostbuild.host_library(m)
    root = [m.root_of(i) for i in range(m.n_dof)]
    mask = np.array([[root[i] != root[j] for j in range(m.n_dof)] for i in range(m.n_dof)])
    for alg, names in (("Minv", ["minv_out"]), ("gradID", ["dq_out", "dqd_out"]),
                       ("gradFD", ["dq_out", "dqd_out"])):
        out = hostbuild.host_eval(lib, m, alg, "f64", g["q"], g["qd"], g["u"])
        for nm in names:
            blocks = out[nm].reshape(-1, m.n_dof, m.n_dof)[:, mask]
            assert np.all(blocks == 0.0)


def test_generation_is_deterministic_and_folds_constants():
    m = models.load("chain7")
    a, fa = codegen.generate_sources(m)
    b, fb = codegen.generate_sources(m)
    assert a == b and fa == fb
    # the model's numbers are literals: no parent tables or inertia arrays in the source
    src = a["k_gradFD_f64_T.cu"] + a["k_gradFD_f64_W.cu"]
    assert "parent" not in src and "[6][6]" not in src
    # fewer flops than the reference program's IR count for gradFD on chain7 (17,131)
    assert fa[("gradFD", "f64")] < 17131


def test_seeded_random_states_match_oracle():
    m = models.load("tree7")
    lib = hostbuild.host_library(m)
    rng = np.random.default_rng(11)
    N, n = 50, m.n_dof
    q, qd, u = rng.uniform(-np.pi, np.pi, (N, n)), rng.uniform(-1, 1, (N, n)), rng.uniform(-1, 1, (N, n))
    for alg in codegen.ALGORITHMS:
        ref = R.evaluate_batch(m, alg, q, qd, u)
        out = hostbuild.host_eval(lib, m, alg, "f64", q, qd, u)
        for nm in ref:
            assert rel_err(out[nm], ref[nm]) < 1e-12


@pytest.mark.parametrize("name", ["chain7", "mixed5", "quad12", "tree7"])
def test_fext_programs_match_reference(name):
    """f_ext (per-link external forces, refdyn.py:79-80) through the generated
    programs vs the reference's outputs with seeded forces (golden 'fext.*')."""
    g = golden(name)
    m = models.load(name)
    lib = hostbuild.host_library(m)
    for alg in codegen.FEXT_ALGORITHMS:
        out = hostbuild.host_eval(lib, m, alg, "f64", g["q"], g["qd"], g["u"], f_ext=g["f_ext"])
        for nm, v in out.items():
            assert rel_err(v, g[f"fext.{alg}.{nm}"]) < TOL["f64"], (name, alg, nm)
