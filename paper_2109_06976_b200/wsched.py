"""Warp-specialised mapping: one CTA = 32 knot points x W warps.

The thread-per-knot mapping (codegen.ptx_body) runs the whole one-knot
program in every thread, so a large robot's live state (hundreds of values
per knot) overflows the register file.  Here the same op list is cut into
the tasks `codegen._Program.run` tags (RNEA sweeps, articulated-inertia
factorisation, one task per Minv column, one per gradient column, ...),
and lane l of EVERY warp works on knot l of the CTA's 32-knot group:

* a task runs on one warp; tasks are levelled by their data dependencies
  into phases separated by CTA barriers, and packed onto warps (LPT) within
  a phase -- independent Minv / gradient columns and independent root trees
  run side by side;
* a value produced in one task and consumed by another goes through an
  arena slot ([slot][lane], one 8-byte word per lane, conflict-free); slots
  are recycled across phases (interval colouring); the arena sits in shared
  memory when it fits, else in an L2-resident global scratch indexed by the
  (persistent) CTA;
* inputs and the sin/cos scratch live in shared memory and joint transforms
  are cheap, so consumers re-materialise them instead of importing them.

Correctness does not depend on the schedule: every task sees exactly the
values the sequential program would, because a consumer only runs in a
later phase than its producers.
"""

from collections import defaultdict

from . import codegen as cg

REMAT = ("in", "xf")
SMEM_BUDGET = 200 * 1024  # bytes of dynamic shared memory per CTA we allow
LANES = 33                # row stride (elements) of every [slot][lane] array


def _srcs(op):
    k = op[0]
    if k == "fma":
        return [a for a in op[2:5] if not isinstance(a, float)]
    if k in ("mul", "add", "sub"):
        return [a for a in op[2:4] if not isinstance(a, float)]
    if k in ("neg", "rcp"):
        return [a for a in op[2:3] if not isinstance(a, float)]
    if k == "st":
        return [a for a in op[3:4] if not isinstance(a, float)]
    return []


def _dsts(op):
    k = op[0]
    if k == "st":
        return []
    if k == "sincos":
        return [op[1], op[2]]
    return [op[1]]


def _remat(tag):
    return tag in REMAT


class Schedule:
    """Tasks, phases, warp assignment and arena slots for one op list."""

    def __init__(self, em, warps):
        self.em = em
        ops, tags = em.ops, em.tasks
        self.def_op = {}
        imported = {}  # reg -> fixed arena slot (split columns: the prefix kernel's exports)
        for i, op in enumerate(ops):
            if op[0] == "imp":
                self.def_op[op[1]] = i
                imported[op[1]] = op[2]
                continue
            for r in _dsts(op):
                self.def_op[r] = i
        self.task_ops = defaultdict(list)
        for i, t in enumerate(tags):
            if not _remat(t) and t != "imp":
                self.task_ops[t].append(i)
        # cross-task values and dependencies
        self.export = {}  # reg -> producing task
        deps = defaultdict(set)
        users = defaultdict(set)
        for t, idxs in self.task_ops.items():
            for i in idxs:
                for r in _srcs(ops[i]):
                    dt = tags[self.def_op[r]]
                    if _remat(dt) or dt == t or dt == "imp":
                        continue
                    self.export[r] = dt
                    deps[t].add(dt)
                    users[r].add(t)
        self.deps = deps
        # levels
        level = {}

        def lv(t):
            if t not in level:
                level[t] = 0 if not deps[t] else 1 + max(lv(d) for d in deps[t])
            return level[t]

        for t in self.task_ops:
            lv(t)
        # sink tasks (nothing depends on them: gradient columns, output-only
        # tasks) go to the last phase, so an early-ready sink (a q-dot column
        # that needs no RNEA at qdd) does not lengthen a middle phase
        if level:
            last = max(level.values())
            has_user = {d for t in self.task_ops for d in deps[t]}
            for t in self.task_ops:
                if t not in has_user:
                    level[t] = last
        self.level = level
        nphase = 1 + max(level.values()) if level else 0
        # cost: arithmetic ops of the task (remat work is small)
        cost = {t: sum(1 for i in idxs if ops[i][0] not in ("st",)) + 1 for t, idxs in self.task_ops.items()}
        self.cost = cost
        self.warps = warps
        self.phases = []
        for p in range(nphase):
            ts = sorted((t for t in self.task_ops if level[t] == p), key=lambda t: (-cost[t], t))
            load = [0] * warps
            assign = [[] for _ in range(warps)]
            for t in ts:
                w = min(range(warps), key=lambda k: (load[k], k))
                assign[w].append(t)
                load[w] += cost[t]
            # keep each warp's tasks in program order (producers before consumers
            # are already in earlier phases; order inside a warp only affects
            # register pressure)
            first = {t: self.task_ops[t][0] for t in ts}
            self.phases.append([sorted(a, key=lambda t: first[t]) for a in assign])
        # arena slots by interval colouring over phases
        iv = []
        for r, t in self.export.items():
            a = level[t]
            b = max(level[u] for u in users[r])
            iv.append((a, b, r))
        iv.sort()
        nimp = 1 + max(imported.values()) if imported else 0
        slot_end = [1 << 30] * nimp  # per slot: last phase it is read in (imports: never recycled)
        self.slot = dict(imported)
        for a, b, r in iv:
            for s, e in enumerate(slot_end):
                if e < a:
                    slot_end[s] = b
                    self.slot[r] = s
                    break
            else:
                self.slot[r] = len(slot_end)
                slot_end.append(b)
        self.nslots = len(slot_end)

    def critical_path(self):
        """Sum over phases of the busiest warp's cost (latency estimate in ops)."""
        return sum(max((sum(self.cost[t] for t in a) for a in ph), default=0) for ph in self.phases)

    def total(self):
        return sum(self.cost.values())


def ptx_block(sched, tasks, dtype, scratch_base, nin_slots, arena_space, out_space, reload_dist=0, ctab=None,
              cta_of=None, my_cta=0):
    """PTX for one warp's tasks in one phase.

    Operands: %0 = this lane's input-staging address (shared, u32),
    %1 = this lane's arena address (shared u32 or global u64),
    %2..%4 = this lane's out0..2 address, %5 = knot valid flag, and over a
    cluster %6 + r = this lane's arena address in CTA rank r (shared::cluster,
    from mapa): a value produced on CTA cta_of[reg] != my_cta is read there.
    Shared [slot][lane] rows are LANES elements apart; a global arena is
    [slot][32 lanes]."""
    em = sched.em
    ops = em.ops
    t = dtype
    es = 8 if t == "f64" else 4
    R = "%%fd" if t == "f64" else "%%f"
    imm = lambda x: cg._imm(x, t)
    lines = []
    consts = {}
    extra = [em.nreg]
    arena_stride = LANES * es if arena_space == "shared" else 32 * es
    out_stride = LANES * es if out_space == "shared" else es
    pred = "@%%p " if out_space == "global" else ""
    sc_pos = {}
    k = 0
    for op in ops:
        if op[0] == "sincos":
            sc_pos[op[1]] = scratch_base + 2 * k
            sc_pos[op[2]] = scratch_base + 2 * k + 1
            k += 1

    def creg(x):
        if x not in consts:
            consts[x] = extra[0]
            extra[0] += 1
            lines.append(f"mov.{t} {R}{consts[x]}, {imm(x)};")
        return f"{R}{consts[x]}"

    have = {}  # reg -> step of last materialisation in this block
    local = set()  # regs computed by this block's own tasks
    step = [0]

    def need(r):
        """Make register r available in this block; returns its name."""
        d = sched.def_op[r]
        dop = ops[d]
        tag = em.tasks[d]
        if r in have:
            reloadable = dop[0] in ("ld", "sincos") or (r in sched.slot and r not in local)
            if not (reload_dist and reloadable and step[0] - have[r] > reload_dist):
                return f"{R}{r}"
        if dop[0] == "ld":
            lines.append(f"ld.shared.{t} {R}{r}, [%0+{dop[2] * LANES * es}];")
        elif dop[0] == "sincos":
            lines.append(f"ld.shared.{t} {R}{r}, [%0+{sc_pos[r] * LANES * es}];")
        elif tag in REMAT:
            emit(dop)
        elif r in sched.slot:
            if cta_of is not None and cta_of.get(r, my_cta) != my_cta:
                lines.append(f"ld.shared::cluster.{t} {R}{r}, [%{6 + cta_of[r]}+{sched.slot[r] * arena_stride}];")
            else:
                lines.append(f"ld.{arena_space}.{t} {R}{r}, [%1+{sched.slot[r] * arena_stride}];")
        else:
            raise cg.GenerationError(f"register {r} used before its definition in task order")
        have[r] = step[0]
        return f"{R}{r}"

    def fresh():
        extra[0] += 1
        return f"{R}{extra[0] - 1}"

    def use(a):
        if isinstance(a, float):
            return ctab.operand(a, lines, fresh) if ctab is not None else imm(a)
        return need(a)

    def emit(op):
        k = op[0]
        step[0] += 1
        if k == "fma":
            a, b, c = op[2], op[3], op[4]
            if isinstance(a, float):
                a, b = b, a
            lines.append(f"fma.rn.{t} {R}{op[1]}, {use(a)}, {use(b)}, {use(c)};")
        elif k in ("mul", "add"):
            a, b = op[2], op[3]
            if isinstance(a, float):
                a, b = b, a
            lines.append(f"{k}.rn.{t} {R}{op[1]}, {use(a)}, {use(b)};")
        elif k == "sub":
            if isinstance(op[2], float):
                lines.append(f"neg.{t} {R}{op[1]}, {use(op[3])};")
                lines.append(f"add.rn.{t} {R}{op[1]}, {R}{op[1]}, {imm(op[2])};")
            else:
                lines.append(f"sub.rn.{t} {R}{op[1]}, {use(op[2])}, {use(op[3])};")
        elif k == "neg":
            lines.append(f"neg.{t} {R}{op[1]}, {use(op[2])};")
        elif k == "rcp":
            lines.append(f"rcp.rn.{t} {R}{op[1]}, {use(op[2])};")
        elif k == "st":
            v = creg(op[3]) if isinstance(op[3], float) else use(op[3])
            lines.append(f"{pred}st.{out_space}.{t} [%{2 + op[1]}+{op[2] * out_stride}], {v};")
            return
        elif k in ("ld", "sincos"):
            return
        else:
            raise cg.GenerationError(f"unknown op {k}")
        have[op[1]] = step[0]
        if em.tasks[sched.def_op[op[1]]] not in REMAT:
            local.add(op[1])
        if op[1] in sched.slot:
            lines.append(f"st.{arena_space}.{t} [%1+{sched.slot[op[1]] * arena_stride}], {R}{op[1]};")

    for task in tasks:
        for i in sched.task_ops[task]:
            op = ops[i]
            if op[0] in ("ld", "sincos"):
                continue
            emit(op)
    head = [f".reg .{t} {R}<{extra[0]}>;"]
    if out_space == "global":
        head += [".reg .pred %%p;", "setp.ne.u32 %%p, %5, 0;"]
    return head + lines


def variant_programs(model, alg, dtype, k, fext=False):
    """Split one knot's program over CTA rows ("variants", blockIdx.y) so a
    small batch spreads over more SMs: one variant per root tree (independent
    sub-programs), and a tree's gradient columns cut into contiguous groups,
    about k groups over the whole robot in proportion to tree size; each
    variant re-computes its tree's prefix (RNEA, Minv, FD) itself.  Every
    variant reads the whole staged input row (full window) so all CTA rows
    share one staging layout and sin/cos table.  Entries no variant stores
    (cross-tree structural zeros) are stored as 0 by the variants, round
    robin.  Returns the list of op lists (`_Emit`)."""
    n = model.n_dof
    trees = [model.subtree(r) for r in model.roots()]
    grad = alg in ("gradID", "gradFD")
    progs = []
    for t, tree in enumerate(trees):
        groups = [None]
        if grad:
            g = max(1, min(len(tree), int(round(k * len(tree) / n))))
            groups = [tree[i * len(tree) // g:(i + 1) * len(tree) // g] for i in range(g)]
        for cols in groups:
            progs.append(cg.generate_knot(model, alg, dtype, trees=(t,), zero_fill=False, cols=cols, fext=fext,
                                          full_window=True))
    if alg in ("Minv", "gradID", "gradFD"):
        stored = {(op[1], op[2]) for em in progs for op in em.ops if op[0] == "st"}
        outs = (0,) if alg == "Minv" else (0, 1)
        zeros = [(o, idx) for o in outs for idx in range(n * n) if (o, idx) not in stored]
        for z, (o, idx) in enumerate(zeros):
            em = progs[z % len(progs)]
            em.ops.append(("st", o, idx, 0.0))
            em.tasks.append("zeros")
    return progs


def split_programs(model, alg, dtype, k, big_tree=0):
    """Small-batch split of a gradient program (two warp-specialised
    launches): kernel A runs the big tree's prefix (RNEA, articulated
    inertias, Minv, FD, RNEA at qdd) once per knot group and stores the values
    the gradient columns import as its output 0 (a [N][nx] scratch) and the
    tree's qdd as output 1; kernel B's CTA-row variants are the big tree's
    gradient columns in ~k groups -- the scratch is their 4th input, so an
    import is an ordinary (re-materialised) load of the staged row -- plus
    the other root trees' whole programs.  All of B's variants share one
    input layout (q, qd, u, scratch) and sin/cos table; cross-tree zeros are
    stored round robin.  Returns (prefix em, [variant ems], nx)."""
    n = model.n_dof
    trees = [model.subtree(r) for r in model.roots()]
    em = cg.generate_knot(model, alg, dtype, trees=(big_tree,), zero_fill=False, full_window=True)
    pre, cols, nx = cg.split_columns(em)
    # prefix: exports -> output 0 (scratch), qdd (gradFD output 2) -> output 1
    pops, ptasks = [], []
    for op, t in zip(pre.ops, pre.tasks):
        if op[0] == "xst":
            op = ("st", 0, op[1], op[2])
        elif op[0] == "st":
            if op[1] != 2:
                raise cg.GenerationError("split prefix stores only qdd")
            op = ("st", 1, op[2], op[3])
        pops.append(op)
        ptasks.append(t)
    prefix = cg._sub_emit(pre, pops, ptasks)

    def with_scratch_input(e):
        """append the scratch row as the 4th input (after u); sin/cos follow it"""
        e.in_layout = list(e.in_layout) + [("x", e.in_total, nx, 0, nx)]
        e.in_total = e.in_total + nx
        return e

    base = em.in_total  # the scratch row starts after q, qd, u
    gtasks = list(dict.fromkeys(t for t in cols.tasks if t.startswith("grad.")))
    g = max(1, min(int(k), len(gtasks)))
    # LPT: column tasks by op count onto the least-loaded group (a column's
    # cost grows with its subtree: column 0 of the torso spans every frame)
    cost = {t: 0 for t in gtasks}
    for t in cols.tasks:
        if t in cost:
            cost[t] += 1
    groups, load = [set() for _ in range(g)], [0] * g
    for t in sorted(gtasks, key=lambda x: (-cost[x], x)):
        j = min(range(g), key=lambda i: (load[i], i))
        groups[j].add(t)
        load[j] += cost[t]
    variants = []
    for grp in groups:
        ops, tasks = [], []
        for op, t in zip(cols.ops, cols.tasks):
            if op[0] == "imp":
                ops.append(("ld", op[1], base + op[2]))
                tasks.append("in")
            elif t in ("in", "xf") or t in grp:
                ops.append(op)
                tasks.append(t)
        variants.append(with_scratch_input(cg._sub_emit(cols, ops, tasks)))
    for t in range(len(trees)):
        if t != big_tree:
            variants.append(with_scratch_input(cg.generate_knot(model, alg, dtype, trees=(t,), zero_fill=False,
                                                                full_window=True)))
    stored = {(op[1], op[2]) for e in variants for op in e.ops if op[0] == "st"}
    zeros = [(o, idx) for o in (0, 1) for idx in range(n * n) if (o, idx) not in stored]
    for z, (o, idx) in enumerate(zeros):
        e = variants[z % len(variants)]
        e.ops.append(("st", o, idx, 0.0))
        e.tasks.append("zeros")
    return prefix, variants, nx


def plan(model, alg, dtype, warps, trees=None, zero_fill=True, fext=False, em=None, ext=None):
    """Schedule + memory plan of the warp-specialised kernel (ext: output
    extents when they differ from the algorithm's, e.g. a split prefix)."""
    if em is None:
        em = cg.generate_knot(model, alg, dtype, trees, zero_fill, fext=fext)
    sched = Schedule(em, warps)
    imports = any(op[0] == "imp" for op in em.ops)
    n = model.n_dof
    es = 8 if dtype == "f64" else 4
    nin = len(em.in_layout)
    nsc = sum(1 for op in em.ops if op[0] == "sincos")
    if ext is None:
        ext = [e for _, e in cg.outputs(alg, n)]
    ext = list(ext) + [0] * (3 - len(ext))
    sin = em.in_total + 2 * nsc
    row = LANES * es
    sout = sum(ext)
    opts = [(True, True), (True, False), (False, True), (False, False)]  # (arena smem, stage outputs)
    if cg.tuning(model, alg, dtype).get("arena") == "global" or imports:
        opts = [(False, True), (False, False)]
    for ar, st in opts:
        smem = row * (sin + (sched.nslots if ar else 0) + (sout if st else 0))
        if smem <= SMEM_BUDGET:
            break
    return dict(em=em, sched=sched, n=n, nin=nin, nsc=nsc, ext=ext, sin=sin, sout=sout,
                arena_smem=ar, stage=st, smem=smem, es=es, warps=warps, imports=imports)
