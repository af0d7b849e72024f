"""The exact PTX the generator emits for the device, executed on CPU by a
small interpreter (tests/support/ptxsim.py), against the reference outputs:
both kernel mappings (thread-per-knot, warp-specialised schedule with its
arena-slot recycling), so scheduling / slot-reuse / re-materialisation bugs
surface without a GPU."""
import math

import numpy as np
import pytest

from conftest import golden, rel_err
from paper_2109_06976_b200 import codegen, models, wsched
from support import ptxsim


def _inputs(g, alg, k, n):
    names = codegen.INPUTS[alg]
    return np.concatenate([g[{"q": "q", "qd": "qd"}.get(nm, "u")][k] for nm in names])


def _sincos_slots(em):
    return [op[3] for op in em.ops if op[0] == "sincos"]


def run_thread(model, alg, dt, x, stage, budget=None, park=False, fext=False, trow=False, hot=0):
    em = codegen.generate_knot(model, alg, dt, fext=fext)
    n = model.n_dof
    nin = em.in_total // n
    ctab = codegen.ConstTable("K", dt)
    plan = None
    nsc = len(_sincos_slots(em))
    if budget:
        plan = codegen.SpillPlan(em, budget, codegen.row_homes(em, nin * n), nin * n + 2 * nsc,
                                 park_outputs=park)
    lines, sc = codegen.ptx_body(em, nin * n, "shared" if stage else "global", ctab=ctab, plan=plan,
                                 trow=trow, row_base=nin * n + 2 * nsc, hot_consts=hot)
    if hot and dt == "f64":
        assert any("%%hc" in ln for ln in lines)
    if trow:
        assert sum("tcgen05.ld" in ln for ln in lines) > 0 and not any("st.shared.f" in ln and "%0+" in ln
                                                                       for ln in lines)
    es = 8 if dt == "f64" else 4
    row = {i: float(v) for i, v in enumerate(x)}
    for k, slot in enumerate(sc):
        row[nin * n + 2 * k] = math.sin(x[slot])
        row[nin * n + 2 * k + 1] = math.cos(x[slot])
    outs = [dict() for _ in range(3)]
    ptxsim.run_block(lines, [row] + outs + [None, None, {}], [es] * 5 + [8, 1], f32=(dt == "f32"),
                     consts={"K": sorted(ctab.index, key=ctab.index.get)})
    if park:  # the kernel's write-back: parked row slots, structural zeros
        for (k, idx), sl in plan.outslot.items():
            outs[k][idx] = row[sl]
        for (k, idx), v in plan.outconst.items():
            outs[k][idx] = v
    return [np.array([o.get(i, np.nan) for i in range(e)]) for o, (_, e) in zip(outs, codegen.outputs(alg, n))]


def run_ws(model, alg, dt, x, warps, arena_space="shared", out_space="shared", fext=False, em=None, outs=None):
    P = wsched.plan(model, alg, dt, warps, fext=fext, em=em)
    S = P["sched"]
    n = P["n"]
    base = P["em"].in_total  # inputs (3 or 4 arrays, or f_ext) then sin/cos
    es = 8 if dt == "f64" else 4
    L = wsched.LANES
    row = {i: float(v) for i, v in enumerate(x)}
    for k, slot in enumerate(_sincos_slots(P["em"])):
        row[base + 2 * k] = math.sin(x[slot])
        row[base + 2 * k + 1] = math.cos(x[slot])
    arena = {}
    outs = [dict() for _ in range(3)] if outs is None else outs
    astride = L * es if arena_space == "shared" else 32 * es
    ostride = L * es if out_space == "shared" else es
    ctab = codegen.ConstTable("K", dt)
    for phase in S.phases:
        for tasks in phase:
            if tasks:
                lines = wsched.ptx_block(S, tasks, dt, base, base, arena_space, out_space, 0, ctab)
                ptxsim.run_block(lines, [row, arena] + outs + [None], [L * es, astride, ostride, ostride, ostride],
                                 f32=(dt == "f32"), consts={"K": sorted(ctab.index, key=ctab.index.get)})
    return [np.array([o.get(i, np.nan) for i in range(e)]) for o, (_, e) in zip(outs, codegen.outputs(alg, n))], S


@pytest.mark.parametrize("name", ["pendulum2", "chain7", "tree7", "mixed5", "quad12"])
@pytest.mark.parametrize("mapping", ["thread", "thread_ra", "thread_park", "thread_trow", "thread_hot", "ws"])
def test_device_ptx_matches_reference(name, mapping):
    g = golden(name)
    m = models.load(name)
    n = m.n_dof
    for alg in codegen.ALGORITHMS:
        for k in (0, 5):
            x = _inputs(g, alg, k, n)
            if mapping == "thread":
                outs = run_thread(m, alg, "f64", x, stage=(k == 0))
            elif mapping == "thread_park":
                # the product layout: outputs parked in the row, written back by map
                outs = run_thread(m, alg, "f64", x, stage=False, budget=16 if k == 0 else 119, park=True)
            elif mapping == "thread_trow":
                # the row in tensor memory (inputs copied in, spills / reloads as tcgen05.st / ld)
                outs = run_thread(m, alg, "f64", x, stage=True, budget=12 if k == 0 else 40, trow=True)
            elif mapping == "thread_hot":
                # the most used table constants held in registers (hot_consts)
                outs = run_thread(m, alg, "f64", x, stage=True, budget=12 if k == 0 else 40, trow=True,
                                  hot=8 if k == 0 else 64)
            elif mapping == "thread_ra":
                # tight register budgets force heavy parking / slot reuse
                outs = run_thread(m, alg, "f64", x, stage=(k == 0), budget=12 if k == 0 else 40)
            else:
                outs, _ = run_ws(m, alg, "f64", x, warps=4 if k == 0 else 7,
                                 arena_space="shared" if k == 0 else "global",
                                 out_space="global" if k == 0 else "shared")
            for (nm, _), o in zip(codegen.outputs(alg, n), outs):
                ref = g[f"{alg}.{nm}"][k:k + 1]
                assert np.all(np.isfinite(o)), (name, alg, nm, "unwritten output")
                assert rel_err(o[None], ref) < 1e-12, (name, alg, nm)


@pytest.mark.parametrize("name,k", [("chain7", 4), ("quad12", 4), ("tree7", 3), ("mixed5", 3), ("humanoid30", 8)])
def test_ws_variants_compose_to_the_whole(name, k):
    """CTA-row variants (wsched.variant_programs): each variant runs on its
    own arena; together they write every output element exactly once and
    match the reference (cross-tree zeros included)."""
    g = golden(name)
    m = models.load(name)
    n = m.n_dof
    for alg in codegen.ALGORITHMS:
        progs = wsched.variant_programs(m, alg, "f64", k)
        if alg in ("gradID", "gradFD"):
            assert len(progs) >= min(k, n) or len(progs) >= len(m.roots())
        stores = [(op[1], op[2]) for em in progs for op in em.ops if op[0] == "st"]
        assert len(stores) == len(set(stores)), (name, alg, "an element is written by two variants")
        x = _inputs(g, alg, 3, n)
        outs = [dict() for _ in range(3)]
        for em in progs:
            run_ws(m, alg, "f64", x, 5, arena_space="shared", out_space="global", em=em, outs=outs)
        for (nm, e), o in zip(codegen.outputs(alg, n), outs):
            got = np.array([o.get(i, np.nan) for i in range(e)])
            assert np.all(np.isfinite(got)), (name, alg, nm, "unwritten output")
            assert rel_err(got[None], g[f"{alg}.{nm}"][3:4]) < 1e-12, (name, alg, nm)


@pytest.mark.parametrize("name,C", [("chain7", 4), ("quad12", 2), ("mixed5", 3), ("humanoid30", 4)])
def test_ws_cluster_arena(name, C):
    """Cluster mapping: tasks over C CTAs x W warps; each value lives in the
    arena of the CTA whose warp produced it, a consumer on another CTA reads
    it with ld.shared::cluster through that CTA's operand (%6 + rank)."""
    g = golden(name)
    m = models.load(name)
    n = m.n_dof
    W = 4
    L = wsched.LANES
    for alg in codegen.ALGORITHMS:
        P = wsched.plan(m, alg, "f64", W * C)
        S, em = P["sched"], P["em"]
        x = _inputs(g, alg, 1, n)
        nin = em.in_total // n
        row = {i: float(v) for i, v in enumerate(x)}
        for k, slot in enumerate(_sincos_slots(em)):
            row[nin * n + 2 * k] = math.sin(x[slot])
            row[nin * n + 2 * k + 1] = math.cos(x[slot])
        wof = {t: w for ph in S.phases for w, ts in enumerate(ph) for t in ts}
        cta_of = {r: wof[t] // W for r, t in S.export.items()}
        arenas = [dict() for _ in range(C)]
        outs = [dict() for _ in range(3)]
        ctab = codegen.ConstTable("K", "f64")
        remote = 0
        for phase in S.phases:
            for w, tasks in enumerate(phase):
                if not tasks:
                    continue
                lines = wsched.ptx_block(S, tasks, "f64", nin * n, nin * n, "shared", "global", 0, ctab,
                                         cta_of=cta_of, my_cta=w // W)
                remote += sum("shared::cluster" in ln for ln in lines)
                ptxsim.run_block(lines, [row, arenas[w // W]] + outs + [None] + arenas,
                                 [L * 8, L * 8, 8, 8, 8, None] + [L * 8] * C,
                                 consts={"K": sorted(ctab.index, key=ctab.index.get)})
        if alg in ("gradFD", "gradID", "Minv"):
            assert remote > 0, (name, alg, "no value crossed CTAs")
        for (nm, e), o in zip(codegen.outputs(alg, n), outs):
            got = np.array([o.get(i, np.nan) for i in range(e)])
            assert np.all(np.isfinite(got)), (name, alg, nm, "unwritten output")
            assert rel_err(got[None], g[f"{alg}.{nm}"][1:2]) < 1e-12, (name, alg, nm)


@pytest.mark.parametrize("name,alg", [("humanoid30", "gradFD"), ("humanoid30", "gradID"), ("quad12", "gradFD")])
def test_ws_split_programs(name, alg):
    """Small-batch split: the prefix program's outputs (the [nx] export row
    and the tree's qdd) feed the column variants as their 4th input; with
    the other trees' variants they write every output element once and match
    the reference."""
    g = golden(name)
    m = models.load(name)
    n = m.n_dof
    pre, progs, nx = wsched.split_programs(m, alg, "f64", 4)
    x = _inputs(g, alg, 2, n)
    scratch, outs = {}, [dict() for _ in range(3)]
    pouts = [scratch, outs[2], {}]  # prefix: output 0 = exports, output 1 = qdd
    run_ws(m, alg, "f64", x, 6, out_space="global", em=pre, outs=pouts)
    assert len(scratch) == nx
    stores = [(op[1], op[2]) for e in progs for op in e.ops if op[0] == "st"]
    assert len(stores) == len(set(stores))
    xs = np.concatenate([x, [scratch[i] for i in range(nx)]])
    for e in progs:
        assert len(e.in_layout) == 4
        run_ws(m, alg, "f64", xs, 5, out_space="global", em=e, outs=outs)
    for (nm, e), o in zip(codegen.outputs(alg, n), outs):
        got = np.array([o.get(i, np.nan) for i in range(e)])
        assert np.all(np.isfinite(got)), (name, alg, nm, "unwritten output")
        assert rel_err(got[None], g[f"{alg}.{nm}"][2:3]) < 1e-12, (name, alg, nm)


@pytest.mark.parametrize("name,trees", [("humanoid30", (1,)), ("humanoid30", (2,)), ("quad12", (3,))])
def test_part_program_with_tmem_row(name, trees):
    """A part program (one root tree of several) with its row in TMEM and its
    outputs staged densely: every element it stores lands at its dense slot,
    and the element map puts it back where the reference has it."""
    g = golden(name)
    m = models.load(name)
    n = m.n_dof
    em = codegen.generate_knot(m, "gradFD", "f64", trees=trees, zero_fill=False)
    L = codegen._layout(m, "gradFD", "f64", em, over={"tmem_row": True})
    assert L.get("trow") and L.get("tpart"), "the part should take the TMEM-row layout"
    ctab = codegen.ConstTable("K", "f64")
    lines, sc = codegen.ptx_body(em, em.in_total, "shared", ctab=ctab, plan=L["plan"], trow=True,
                                 row_base=L["sin"], dense=L["dense"])
    k = 2
    x_full = _inputs(g, "gradFD", k, n)
    lo, np_ = em.lo, em.np
    x = np.concatenate([x_full[a * n + lo:a * n + lo + np_] for a in range(3)])
    row = {i: float(v) for i, v in enumerate(x)}
    for j, slot in enumerate(sc):
        row[em.in_total + 2 * j] = math.sin(x[slot])
        row[em.in_total + 2 * j + 1] = math.cos(x[slot])
    staged = {}
    ptxsim.run_block(lines, [row, staged, {}, {}, None, None, {}], [8, 8, 8, 8, 8, 8, 1],
                     consts={"K": sorted(ctab.index, key=ctab.index.get)})
    assert len(staged) == len(L["tpart"])
    ext = [e for _, e in codegen.outputs("gradFD", n)]
    ref = np.concatenate([g[f"gradFD.{nm}"][k] for nm, _ in codegen.outputs("gradFD", n)])
    got = np.array([staged[j] for j in range(len(L["tpart"]))])
    want = ref[np.array(L["tpart"])]
    assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, np.max(np.abs(ref))), (name, trees)
    assert sum(ext) > len(L["tpart"])


@pytest.mark.parametrize("alg", ["gradFD", "gradID", "Minv"])
def test_tmem_row_zero_map(alg):
    """quad12's whole program on the TMEM row with its structural zeros not
    staged (trow_zmap): the program stages only the non-zero outputs, and the
    write-back's element map (dense slot or -1 = 0) rebuilds every output
    element the reference has, cross-leg zeros included."""
    name = "quad12"
    g = golden(name)
    m = models.load(name)
    n = m.n_dof
    em = codegen.generate_knot(m, alg, "f64")
    L = codegen._layout(m, alg, "f64", em, over={"tmem_row": True, "trow_zmap": True})
    assert L.get("trow") and L.get("zmap") and not L.get("tpart")
    zmap = L["zmap"]
    ext = [e for _, e in codegen.outputs(alg, n)]
    assert len(zmap) == sum(ext) and 0 < sum(j >= 0 for j in zmap) < len(zmap)
    ctab = codegen.ConstTable("K", "f64")
    lines, sc = codegen.ptx_body(em, em.in_total, "shared", ctab=ctab, plan=L["plan"], trow=True,
                                 row_base=L["sin"], dense=L["dense"])
    k = 1
    x = _inputs(g, alg, k, n)
    row = {i: 0.0 for i in range(L["sin"])}  # the odd-stride pad slot is copied too
    row.update({i: float(v) for i, v in enumerate(x)})
    for j, slot in enumerate(sc):
        row[em.in_total + 2 * j] = math.sin(x[slot])
        row[em.in_total + 2 * j + 1] = math.cos(x[slot])
    staged = {}
    ptxsim.run_block(lines, [row, staged, {}, {}, None, None, {}], [8, 8, 8, 8, 8, 8, 1],
                     consts={"K": sorted(ctab.index, key=ctab.index.get)})
    assert sorted(staged) == sorted(j for j in zmap if j >= 0)
    got = np.array([staged[j] if j >= 0 else 0.0 for j in zmap])
    ref = np.concatenate([g[f"{alg}.{nm}"][k].ravel() for nm, _ in codegen.outputs(alg, n)])
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref))), alg
    assert np.all(ref[np.array(zmap) < 0] == 0.0)


def test_ws_schedule_properties():
    m = models.load("humanoid30")
    P = wsched.plan(m, "gradFD", "f64", 16)
    S = P["sched"]
    # every dependency points to an earlier phase
    for t, ds in S.deps.items():
        assert all(S.level[d] < S.level[t] for d in ds)
    # the three independent trees' gradient columns run concurrently
    assert S.critical_path() < S.total() / 4
    # slot recycling keeps the arena well below one slot per exported value
    assert S.nslots < len(S.export)


def test_ws_humanoid30_gradfd_one_knot():
    g = golden("humanoid30")
    m = models.load("humanoid30")
    x = _inputs(g, "gradFD", 2, m.n_dof)
    outs, _ = run_ws(m, "gradFD", "f64", x, warps=16, arena_space="global", out_space="global")
    for (nm, _), o in zip(codegen.outputs("gradFD", m.n_dof), outs):
        assert rel_err(o[None], g[f"gradFD.{nm}"][2:3]) < 1e-12


def _run_part(model, alg, x_full, trees, zero_fill, budget):
    """One part program (a subset of root trees, inputs from its dof window),
    as the large-batch kernel runs it: planned registers, parked outputs."""
    em = codegen.generate_knot(model, alg, "f64", trees, zero_fill)
    n = model.n_dof
    nin = len(codegen.INPUTS[alg])
    lo, np_ = em.lo, em.np
    x = np.concatenate([x_full[a * n + lo:a * n + lo + np_] for a in range(nin)])
    nsc = len(_sincos_slots(em))
    plan = codegen.SpillPlan(em, budget, codegen.row_homes(em, nin * np_), nin * np_ + 2 * nsc, park_outputs=True)
    ctab = codegen.ConstTable("K", "f64")
    lines, sc = codegen.ptx_body(em, nin * np_, "global", ctab=ctab, plan=plan)
    row = {i: float(v) for i, v in enumerate(x)}
    for k, slot in enumerate(sc):
        row[nin * np_ + 2 * k] = math.sin(x[slot])
        row[nin * np_ + 2 * k + 1] = math.cos(x[slot])
    ptxsim.run_block(lines, [row, {}, {}, {}, None], [8] * 5, consts={"K": sorted(ctab.index, key=ctab.index.get)})
    outs = [dict() for _ in range(3)]
    for (k, idx), sl in plan.outslot.items():
        outs[k][idx] = row[sl]
    for (k, idx), v in plan.outconst.items():
        outs[k][idx] = v
    return outs


@pytest.mark.parametrize("name", ["quad12", "humanoid30"])
def test_part_programs_compose_to_the_whole(name):
    """The large-batch path runs one program per root tree (part 0 also
    writes the cross-part zeros); together they must reproduce the reference
    exactly, each part touching only its own output elements."""
    g = golden(name)
    m = models.load(name)
    n = m.n_dof
    trees = list(range(len(m.roots())))
    for alg in ("FD", "gradFD") if name == "humanoid30" else codegen.ALGORITHMS:
        x = _inputs(g, alg, 1, n)
        merged = [dict() for _ in range(3)]
        for t in trees:
            if name == "humanoid30" and t == 0 and alg == "gradFD":
                continue  # the torso part runs warp-specialised (covered on the GPU)
            outs = _run_part(m, alg, x, (t,), t == 0, 64)
            owned = set(m.subtree(m.roots()[t]))
            for k, o in enumerate(outs):
                for idx, v in o.items():
                    # only part 0's structural zeros may be overwritten (the parts run in order)
                    assert idx not in merged[k] or merged[k][idx] == 0.0, (alg, t, k, idx)
                    if len(o) and codegen.outputs(alg, n)[k][1] == n * n and v != 0.0:
                        assert idx // n in owned and idx % n in owned
                    merged[k][idx] = v
        for (nm, e), o in zip(codegen.outputs(alg, n), merged):
            ref = g[f"{alg}.{nm}"][1]
            got = np.array([o.get(i, np.nan) for i in range(e)])
            if name == "humanoid30" and alg == "gradFD":
                own = [i for i in range(e) if not np.isnan(got[i])]
                assert rel_err(got[own][None], ref[own][None]) < 1e-12, (name, alg, nm)
            else:
                assert np.all(np.isfinite(got)), (name, alg, nm)
                assert rel_err(got[None], ref[None]) < 1e-12, (name, alg, nm)


def test_spill_plan_invariants():
    """Register plan, replayed op by op: a reload finds its own value in the
    slot, a slot is only overwritten once its previous value is dead, parked
    outputs are never overwritten, slots are recycled, and a tighter budget
    costs more reloads."""
    m = models.load("chain7")
    em = codegen.generate_knot(m, "gradFD", "f64")
    homes = codegen.row_homes(em, 21)
    last = {}
    for i, op in enumerate(em.ops):
        for r in codegen.op_srcs(op):
            last[r] = i
    for budget, pf in ((8, None), (40, None), (119, None), (24, (32, 4)), (96, (96, 12))):
        plan = codegen.SpillPlan(em, budget, homes, 35, park_outputs=True, prefetch=pf)
        owner = {sl: v for v, sl in homes.items()}
        for i, op in enumerate(em.ops):
            for a in plan.before.get(i, ()):
                assert owner.get(plan.slot[a]) == a, (budget, i, a)
            if op[0] == "st" and not isinstance(op[3], float):
                sl = plan.outslot[(op[1], op[2])]
                prev = owner.get(sl)
                assert prev is None or (not isinstance(prev, tuple) and last.get(prev, -1) < i), (budget, i, prev)
                owner[sl] = ("out", op[1], op[2])
            for v, sl in plan.after.get(i, ()):
                prev = owner.get(sl)
                assert prev is None or (not isinstance(prev, tuple) and last.get(prev, -1) <= i), (budget, i, prev)
                owner[sl] = v
        parked = {v for v in owner.values() if isinstance(v, tuple)}
        assert len(parked) == len(plan.outslot)
        assert plan.nslots < 35 + plan.stores + len(plan.outslot)  # slots were recycled
    tight = codegen.SpillPlan(em, 8, homes, 35)
    loose = codegen.SpillPlan(em, 119, homes, 35)
    assert tight.reloads > loose.reloads and loose.stores <= tight.stores


@pytest.mark.parametrize("name", ["chain7", "quad12", "mixed5"])
@pytest.mark.parametrize("mapping", ["thread_park", "ws"])
def test_device_ptx_with_fext(name, mapping):
    """The f_ext kernels' PTX (f_ext staged after q, qd, u in the knot's row)
    against the reference's outputs with seeded external forces."""
    g = golden(name)
    m = models.load(name)
    n = m.n_dof
    for alg in codegen.FEXT_ALGORITHMS:
        x = np.concatenate([_inputs(g, alg, 3, n), g["f_ext"][3].ravel()])
        if mapping == "thread_park":
            outs = run_thread(m, alg, "f64", x, stage=False, budget=40, park=True, fext=True)
        else:
            outs, _ = run_ws(m, alg, "f64", x, warps=5, arena_space="global", out_space="global", fext=True)
        for (nm, _), o in zip(codegen.outputs(alg, n), outs):
            assert rel_err(o[None], g[f"fext.{alg}.{nm}"][3:4]) < 1e-12, (name, alg, nm)


@pytest.mark.parametrize("name,trees", [("humanoid30", (0,)), ("chain7", None), ("quad12", None)])
@pytest.mark.parametrize("alg", ["gradID", "gradFD"])
def test_split_prefix_and_columns(name, trees, alg):
    """Split gradient program (large root trees): the prefix kernel's PTX
    (register plan, exports stored to the knot's scratch slots) followed by
    the one-phase column kernel's PTX (imports read from that scratch as its
    arena) reproduces the reference."""
    g = golden(name)
    m = models.load(name)
    n = m.n_dof
    k = 4
    em = codegen.generate_knot(m, alg, "f64", trees, trees is None, lowmem=True)
    pre, cols, nx = codegen.split_columns(em)
    lo, np_ = em.lo, em.np
    x_full = _inputs(g, alg, k, n)
    x = np.concatenate([x_full[a * n + lo:a * n + lo + np_] for a in range(3)])
    # prefix: thread-per-knot with its register plan
    nsc = len(_sincos_slots(pre))
    plan = codegen.SpillPlan(pre, 48, codegen.row_homes(pre, pre.in_total), pre.in_total + 2 * nsc, park_outputs=True)
    ctab = codegen.ConstTable("K", "f64")
    lines, sc = codegen.ptx_body(pre, pre.in_total, "global", ctab=ctab, plan=plan)
    row = {i: float(v) for i, v in enumerate(x)}
    for j, slot in enumerate(sc):
        row[pre.in_total + 2 * j] = math.sin(x[slot])
        row[pre.in_total + 2 * j + 1] = math.cos(x[slot])
    scratch = {}
    ptxsim.run_block(lines, [row, {}, {}, {}, None, scratch], [8, 8, 8, 8, 8, 32 * 8],
                     consts={"K": sorted(ctab.index, key=ctab.index.get)})
    assert len(scratch) == nx
    outs = [dict() for _ in range(3)]
    for (kk, idx), sl in plan.outslot.items():
        outs[kk][idx] = row[sl]
    for (kk, idx), v in plan.outconst.items():
        outs[kk][idx] = v
    # columns, thread-per-knot: imports reloaded from the scratch, prefetched
    cplan = codegen.SpillPlan(cols, 40, codegen.row_homes(cols, cols.in_total),
                              cols.in_total + 2 * len(_sincos_slots(cols)), prefetch=(48, 6))
    ctab = codegen.ConstTable("K", "f64")
    lines, sc = codegen.ptx_body(cols, cols.in_total, "global", ctab=ctab, plan=cplan)
    crow = {i: float(v) for i, v in enumerate(x)}
    for j, slot in enumerate(sc):
        crow[cols.in_total + 2 * j] = math.sin(x[slot])
        crow[cols.in_total + 2 * j + 1] = math.cos(x[slot])
    touts = [dict(o) for o in outs]
    ptxsim.run_block(lines, [crow] + touts + [None, dict(scratch)], [8, 8, 8, 8, 8, 32 * 8],
                     consts={"K": sorted(ctab.index, key=ctab.index.get)})
    # the same with the most-reloaded imports homed in tensor memory
    tslot, tcols = codegen.tmem_homes(cplan, 24, 8)
    assert tslot and tcols >= 2 * len(tslot)
    ctab = codegen.ConstTable("K", "f64")
    lines, sc = codegen.ptx_body(cols, cols.in_total, "global", ctab=ctab, plan=cplan, tslot=tslot)
    assert sum("tcgen05.ld" in ln for ln in lines) > 0
    mouts = [dict(o) for o in outs]
    mrow = {i: float(v) for i, v in enumerate(x)}  # a fresh row (the run above recycled input slots)
    for j, slot in enumerate(sc):
        mrow[cols.in_total + 2 * j] = math.sin(x[slot])
        mrow[cols.in_total + 2 * j + 1] = math.cos(x[slot])
    ptxsim.run_block(lines, [mrow] + mouts + [None, dict(scratch), {}], [8, 8, 8, 8, 8, 32 * 8, 1],
                     consts={"K": sorted(ctab.index, key=ctab.index.get)})
    for a, b in zip(mouts, touts):
        assert a == b
    # one program per gradient column (the product kernel's layout): sin/cos
    # exported too, each program reading only what it uses
    pre2, progs, nx2 = codegen.split_columns(em, by_task=True)
    ctab = codegen.ConstTable("K", "f64")
    lines, sc = codegen.ptx_body(pre2, pre2.in_total, "global", ctab=ctab,
                                 plan=codegen.SpillPlan(pre2, 48, codegen.row_homes(pre2, pre2.in_total),
                                                        pre2.in_total + 2 * len(_sincos_slots(pre2)),
                                                        park_outputs=True))
    row2 = {i: float(v) for i, v in enumerate(x)}
    for j, slot in enumerate(sc):
        row2[pre2.in_total + 2 * j] = math.sin(x[slot])
        row2[pre2.in_total + 2 * j + 1] = math.cos(x[slot])
    scratch2 = {}
    ptxsim.run_block(lines, [row2, {}, {}, {}, None, scratch2], [8, 8, 8, 8, 8, 32 * 8],
                     consts={"K": sorted(ctab.index, key=ctab.index.get)})
    assert len(scratch2) == nx2
    pouts = [dict(o) for o in outs]
    for prog in progs:
        assert not any(op[0] == "sincos" for op in prog.ops)
        cp = codegen.SpillPlan(prog, 24, codegen.row_homes(prog, prog.in_total), prog.in_total, prefetch=(32, 4))
        ctab = codegen.ConstTable("K", "f64")
        lines, _ = codegen.ptx_body(prog, prog.in_total, "global", ctab=ctab, plan=cp)
        prow = {i: float(v) for i, v in enumerate(x)}
        ptxsim.run_block(lines, [prow] + pouts + [None, dict(scratch2)], [8, 8, 8, 8, 8, 32 * 8],
                         consts={"K": sorted(ctab.index, key=ctab.index.get)})
    touts = [touts, pouts]
    # columns: one phase, arena = the scratch
    P = wsched.plan(m, alg, "f64", 6, em=cols)
    S = P["sched"]
    assert len(S.phases) == 1 and S.nslots >= nx
    L = wsched.LANES
    srow = {i: float(v) for i, v in enumerate(x)}
    for j, slot in enumerate(_sincos_slots(cols)):
        srow[cols.in_total + 2 * j] = math.sin(x[slot])
        srow[cols.in_total + 2 * j + 1] = math.cos(x[slot])
    ctab = codegen.ConstTable("K", "f64")
    for tasks in S.phases[0]:
        if tasks:
            lines = wsched.ptx_block(S, tasks, "f64", cols.in_total, cols.in_total, "global", "global", 0, ctab)
            ptxsim.run_block(lines, [srow, scratch] + outs + [None], [L * 8, 32 * 8, 8, 8, 8],
                             consts={"K": sorted(ctab.index, key=ctab.index.get)})
    owned = set(range(lo, lo + np_))
    for variant in [outs] + touts:
        for (nm, e), o in zip(codegen.outputs(alg, n), variant):
            ref = g[f"{alg}.{nm}"][k]
            idx = [i for i in range(e) if (i // n in owned and i % n in owned) if e == n * n] or \
                  [i for i in range(e) if i in owned]
            got = np.array([o.get(i, np.nan) for i in idx])
            assert np.all(np.isfinite(got)), (name, alg, nm)
            assert rel_err(got[None], ref[idx][None]) < 1e-12, (name, alg, nm)


def run_fs(model, alg, dt, x, warps, variants, fext=False):
    """The fine-grained mapping (fsched): every (variant, warp) block of the
    exact device PTX, warps interleaved phase by phase (each warp's
    registers persist across its barriers), arena shared by the variant's
    warps; outputs merged over the variants."""
    from paper_2109_06976_b200 import fsched
    em = codegen.generate_knot(model, alg, dt, fext=fext)
    n = model.n_dof
    es = 8 if dt == "f64" else 4
    L = 33
    row = {i: float(v) for i, v in enumerate(x)}
    for k, slot in enumerate(_sincos_slots(em)):
        row[em.in_total + 2 * k] = math.sin(x[slot])
        row[em.in_total + 2 * k + 1] = math.cos(x[slot])
    outs = [dict() for _ in range(3)]
    progs = fsched.split_variants(em, variants) if alg in ("gradID", "gradFD") else [em]
    scheds = []
    for p in progs:
        S = fsched.FineSchedule(p, warps)
        scheds.append(S)
        ctab = codegen.ConstTable("K", dt)
        scs = [op[3] for op in em.ops if op[0] == "sincos"]
        parts = [ptxsim.split_barriers(fsched.ptx_warp(S, w, dt, em.in_total, "global", ctab, sincos_slots=scs))
                 for w in range(warps)]
        assert all(len(pp) == S.nphases for pp in parts)
        arena = {}
        regs = [dict() for _ in range(warps)]
        consts = {"K": sorted(ctab.index, key=ctab.index.get)}
        for ph in range(S.nphases):
            for w in range(warps):
                ptxsim.run_block(parts[w][ph], [row, arena] + outs + [None], [L * es, L * es, es, es, es],
                                 f32=(dt == "f32"), consts=consts, regs=regs[w])
    return [np.array([o.get(i, np.nan) for i in range(e)]) for o, (_, e) in zip(outs, codegen.outputs(alg, n))], scheds


@pytest.mark.parametrize("name", ["pendulum2", "chain7", "tree7", "mixed5", "quad12"])
@pytest.mark.parametrize("alg", ["ID", "Minv", "FD", "gradID", "gradFD"])
def test_fs_schedule_matches_reference(name, alg):
    """Fine-grained schedule (fsched): 8 warps, 3 column variants for the
    gradients -- every variant's blocks run phase by phase against the
    reference outputs; warps read other warps' values only from the arena."""
    g = golden(name)
    m = models.load(name)
    n = m.n_dof
    k = 1
    x = _inputs(g, alg, k, n)
    got, scheds = run_fs(m, alg, "f64", x, 8, 3)
    for (nm, _), v in zip(codegen.outputs(alg, n), got):
        ref = g[f"{alg}.{nm}"][k]
        assert np.all(np.isfinite(v)), (name, alg, nm)
        assert rel_err(v[None], ref[None]) < 1e-12, (name, alg, nm)
