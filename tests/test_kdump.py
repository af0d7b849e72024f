"""The reference's "rbdkernel v1" kernel text (ir.py:161-227) as a wire
format: its own dumps (written with numpy >= 2 constant reprs, which its
loader rejects) ingested, turned into the generator's op list and run -- as
exact device PTX on the CPU here, compiled for sm_100a and batched on the
GPU -- against the reference's outputs; and this generator's programs dumped
in the same format and ingested back."""
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden, rel_err
from paper_2109_06976_b200 import codegen, kdump, models
from support import ptxsim

DUMPS = [("chain7", "gradFD"), ("quad12", "gradID"), ("tree7", "FD"), ("mixed5", "Minv")]


def _text(name, alg):
    with open(os.path.join(GOLDEN, f"rbdkernel_{name}_{alg}.txt")) as fh:
        return fh.read()


def _run_em(em, x, budget=40):
    plan = codegen.SpillPlan(em, budget, codegen.row_homes(em, em.in_total),
                             em.in_total + 2 * sum(1 for op in em.ops if op[0] == "sincos"), park_outputs=True)
    ctab = codegen.ConstTable("K", em.dtype)
    lines, sc = codegen.ptx_body(em, em.in_total, "global", ctab=ctab, plan=plan)
    row = {i: float(v) for i, v in enumerate(x)}
    for j, slot in enumerate(sc):
        row[em.in_total + 2 * j] = math.sin(x[slot])
        row[em.in_total + 2 * j + 1] = math.cos(x[slot])
    ptxsim.run_block(lines, [row, {}, {}, {}, None], [8] * 5, consts={"K": sorted(ctab.index, key=ctab.index.get)})
    outs = [dict() for _ in range(3)]
    for (k, idx), sl in plan.outslot.items():
        outs[k][idx] = row[sl]
    for (k, idx), v in plan.outconst.items():
        outs[k][idx] = v
    return outs


def _x(g, alg, k, n):
    return np.concatenate([g[{"q": "q", "qd": "qd"}.get(nm, "u")][k] for nm in codegen.INPUTS[alg]])


def test_loader_accepts_numpy2_reprs_and_rejects_garbage():
    text = _text("chain7", "gradFD")
    assert "np.float64(" in text  # the reference's own dump under numpy >= 2
    prog = kdump.load_text(text)
    assert prog.meta["algorithm"] == "gradFD" and prog.arena_size == 4650 and len(prog.phases) == 91
    with pytest.raises(kdump.KernelFormatError):
        kdump.load_text("rbdkernel v2\n")
    with pytest.raises(kdump.KernelFormatError):
        kdump.load_text("rbdkernel v1\narena 4\nphase p\nitem\n  frobnicate 1 2\n")


@pytest.mark.parametrize("name,alg", DUMPS)
def test_reference_ir_ingested_matches_reference(name, alg):
    g = golden(name)
    m = models.load(name)
    em = kdump.to_emit(kdump.load_text(_text(name, alg)))
    for k in (0, 7):
        outs = _run_em(em, _x(g, alg, k, m.n_dof))
        for (nm, e), o in zip(codegen.outputs(alg, m.n_dof), outs):
            got = np.array([o.get(i, np.nan) for i in range(e)])
            assert rel_err(got[None], g[f"{alg}.{nm}"][k:k + 1]) < 1e-12, (name, alg, nm)


@pytest.mark.parametrize("name,alg", [("chain7", "gradFD"), ("quad12", "Minv"), ("pendulum2", "ID")])
def test_own_program_dump_round_trip(name, alg):
    g = golden(name)
    m = models.load(name)
    text = kdump.dump_text(m, alg)
    prog = kdump.load_text(text)
    assert prog.meta["generator"] == "paper_2109_06976_b200" and len(prog.phases) >= 2
    outs = _run_em(kdump.to_emit(prog), _x(g, alg, 3, m.n_dof))
    for (nm, e), o in zip(codegen.outputs(alg, m.n_dof), outs):
        got = np.array([o.get(i, np.nan) for i in range(e)])
        assert rel_err(got[None], g[f"{alg}.{nm}"][3:4]) < 1e-12, (name, alg, nm)


@pytest.mark.gpu
@pytest.mark.parametrize("name,alg", DUMPS)
def test_reference_ir_compiled_for_b200(name, alg):
    import ctypes
    import torch
    g = golden(name)
    m = models.load(name)
    so = kdump.compile_program(_text(name, alg), m)
    lib = ctypes.CDLL(so)
    lib.rbd_ingested.argtypes = [ctypes.c_void_p] * 6 + [ctypes.c_int64, ctypes.c_void_p]
    N = 20000  # several CTAs, ragged tail
    reps = -(-N // 16)
    tile = lambda x: np.tile(x, (reps, 1))[:N]
    xs = [torch.from_numpy(tile(g[k])).cuda() for k in ("q", "qd", "u")][:len(codegen.INPUTS[alg])]
    outs = [torch.full((N, e), np.nan, dtype=torch.float64, device="cuda") for _, e in codegen.outputs(alg, m.n_dof)]
    ptr = lambda t: ctypes.c_void_p(t.data_ptr())
    args = [ptr(x) for x in xs] + [None] * (3 - len(xs)) + [ptr(o) for o in outs] + [None] * (3 - len(outs))
    assert lib.rbd_ingested(*args, N, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
    torch.cuda.synchronize()
    for (nm, _), o in zip(codegen.outputs(alg, m.n_dof), outs):
        assert rel_err(o.cpu().numpy(), tile(g[f"{alg}.{nm}"])) < 1e-9, (name, alg, nm)


@pytest.mark.parametrize("mutate,match", [
    (lambda t: "\n".join(l for l in t.splitlines() if not l.startswith(("phase", "item", "  "))), "no phases"),
    (lambda t: t.replace("\narena ", "\narena 1 #", 1), "outside arena"),
])
def test_load_text_validates_like_reference(mutate, match):
    """ir.py:79-99: empty phase lists and out-of-arena segments/slots raise."""
    bad = mutate(_text("tree7", "FD"))
    with pytest.raises(kdump.KernelFormatError, match=match):
        kdump.load_text(bad)


def test_load_text_rejects_out_of_range_slot():
    text = _text("tree7", "FD")
    arena = int(next(l for l in text.splitlines() if l.startswith("arena")).split()[1])
    lines = text.splitlines()
    k = next(i for i, l in enumerate(lines) if l.startswith("  add") or l.startswith("  mul"))
    parts = lines[k].split()
    parts[1] = str(arena + 5)
    lines[k] = "  " + " ".join(parts)
    with pytest.raises(kdump.KernelFormatError, match="outside arena"):
        kdump.load_text("\n".join(lines))
