"""Fine-grained warp-specialised schedule ("fs" mapping): the one-knot op
list -- the generator's DAG, not its coarse tasks -- list-scheduled over the W
warps of a CTA in barrier-separated phases, each warp's whole program one
straight-line block with its values in registers across phases.

Why: with lane = knot (32 knots per warp), a CTA's throughput per SM is the
same whether it holds 1 or 32 live knots, so what bounds a small batch is the
per-knot dependency chain and how evenly one knot's work spreads over the
SM's four schedulers.  The task-level schedule (wsched.Schedule) keeps whole
RNEA sweeps / IA factorisations on one warp (chain7 gradFD: 2,831 of 10,243
ops on its critical path at 8 warps; ID: all 663 on one warp) while the
DAG's own latency-weighted critical path is ~1.5k cycles.

Schedule (critical-path list scheduling under a B200 cost model):

* nodes are the non-rematerialised ops; input loads, sin/cos and joint
  transform entries are re-materialised by each warp that uses them;
* priority = latency-weighted bottom level (longest path to a sink);
* a phase is a time window: an op goes to the warp where it can start first
  (the warp's issue slot and the fp64/fp32 pipe it shares with the other
  warps of its SM sub-partition, wid % 4), preferring the warp that already
  holds its operands; operands produced on ANOTHER warp must come from an
  earlier phase (shared memory, visible after the barrier) and cost a load;
  operands produced on the SAME warp in any phase are registers; an op that
  cannot start within `delta` cycles of the phase start, or whose in-phase
  operands sit on two warps, waits for the next phase;
* phases are separated by `bar.sync 1` inside every warp's block (all warps
  run the same number of barriers); a value read by another warp gets a
  [slot][lane] arena slot in shared memory, recycled by interval colouring;
* (delta, program-order lookahead window) is chosen per program by
  simulating the schedule over a sweep.

Column variants (`split_variants`): for a gradient program, CTA row y
(blockIdx.y) runs the prefix (RNEA, articulated inertias, Minv, FD, RNEA at
qdd) plus only its share of the gradient columns, so a small batch spreads
over C x more SMs; each variant is scheduled on its own.

Correctness does not depend on the schedule: every op runs after its
operands -- earlier in its own warp's block, or on another warp in an
earlier phase (published to shared memory before the barrier).
"""

import heapq
from collections import defaultdict

from . import codegen as cg

REMAT = ("in", "xf")

# B200 cost model (cycles).  DFMA/DADD/DMUL: the fp64 pipe takes a 32-lane
# warp instruction every 2 cycles per SM sub-partition; fp32 every cycle.
# Latencies: dependent fp64 arithmetic ~8, fp32 ~4, rcp.rn (MUFU + Newton
# steps) ~48 / ~20; negations fold into the consumer's operand modifier.
LAT = {"f64": {"fma": 8, "mul": 8, "add": 8, "sub": 8, "neg": 0, "rcp": 48, "st": 0},
       "f32": {"fma": 4, "mul": 4, "add": 4, "sub": 4, "neg": 0, "rcp": 20, "st": 0}}
PIPE = {"f64": 2, "f32": 1}
LDS_LAT = 30      # shared-memory load latency (imports from other warps)
BAR = 40          # barrier release + skew
DELTAS = (80, 160, 320, 640, 1280)
WINDOWS = (600, 2000, 1 << 30)
REMAT_DIST = 400  # re-materialise an input / transform entry whose last copy is older than this
IMPORT_PENALTY = 24  # cycles an extra cross-warp value is worth (arena pressure)


def _is_remat(op, tag):
    return tag in REMAT or op[0] in ("ld", "sincos", "imp")


class FineSchedule:
    """List schedule of an op list over `warps` warps (see module doc)."""

    def __init__(self, em, warps, delta=None, deltas=DELTAS, window=None, windows=WINDOWS, max_slots=None):
        self.em = em
        self.warps = warps
        ops, tags = em.ops, em.tasks
        dt = em.dtype
        self.def_op = {}
        for i, op in enumerate(ops):
            if op[0] == "imp":
                self.def_op[op[1]] = i
                continue
            for r in cg.op_dsts(op):
                self.def_op[r] = i
        nodes = [i for i, op in enumerate(ops) if not _is_remat(op, tags[i])]
        self.nodes = nodes
        preds = {}
        succs = defaultdict(list)
        for i in nodes:
            ps = set()
            for r in cg.op_srcs(ops[i]):
                d = self.def_op[r]
                if not _is_remat(ops[d], tags[d]):
                    ps.add(d)
            preds[i] = sorted(ps)
            for d in ps:
                succs[d].append(i)
        self.preds, self.succs = preds, succs
        lat = LAT[dt]
        self.lat = {i: lat[ops[i][0]] for i in nodes}
        self.cost = {i: (PIPE[dt] if ops[i][0] not in ("neg", "st") else (1 if ops[i][0] == "st" else 0))
                     for i in nodes}
        bl = {}
        for i in reversed(nodes):
            bl[i] = self.lat[i] + max((bl[s] for s in succs[i]), default=0) + self.cost[i]
        self.bl = bl
        self.pos = {v: k for k, v in enumerate(nodes)}
        cands = [(d, w) for d in ((delta,) if delta else deltas) for w in ((window,) if window else windows)]
        best = None
        for d, w in cands:
            r = self._list_schedule(d, w)
            self.est, self.phase_of, self.warp_of, self.order = r
            self._build()
            fits = max_slots is None or self.nslots <= max_slots
            key = (not fits, r[0] if fits else self.nslots)
            if best is None or key < best[0]:
                best = (key, r, d, w)
        _, r, self.delta, self.window = best
        self.est, self.phase_of, self.warp_of, self.order = r
        self._build()

    # -- scheduling -------------------------------------------------------------
    def _list_schedule(self, delta, window):
        W = self.warps
        preds, succs, lat, cost, bl = self.preds, self.succs, self.lat, self.cost, self.bl
        pos, nodes = self.pos, self.nodes
        indeg = {i: len(preds[i]) for i in nodes}
        heap, held = [], []
        done = set()
        lo_ptr = [0]

        def lo():
            while lo_ptr[0] < len(nodes) and nodes[lo_ptr[0]] in done:
                lo_ptr[0] += 1
            return lo_ptr[0]

        def offer(v):
            if pos[v] < lo() + window:
                heapq.heappush(heap, (-bl[v], v))
            else:
                heapq.heappush(held, (pos[v], v))

        for i in nodes:
            if indeg[i] == 0:
                offer(i)
        phase_of, warp_of, finish, order = {}, {}, {}, []
        left = len(nodes)
        t0, p = 0, 0
        rng = range(W)
        while left:
            cur = [t0] * W
            pipe = [t0] * 4
            imported = [set() for _ in rng]
            deferred = []
            placed = 0
            end = t0
            limit = t0 + delta
            while heap:
                if placed and min(cur) > limit:
                    break  # every warp is past the window: close the phase
                _, v = heapq.heappop(heap)
                ready = t0
                w = -1
                split = False
                for u in preds[v]:
                    if phase_of[u] == p:
                        wu = warp_of[u]
                        if w >= 0 and wu != w:
                            split = True
                            break
                        w = wu
                        if finish[u] > ready:
                            ready = finish[u]
                if split:
                    deferred.append(v)
                    continue
                big = cost[v] > 1
                if w < 0:
                    bt = None
                    for k in rng:
                        nimp = 0
                        for u in preds[v]:
                            if warp_of[u] != k and u not in imported[k]:
                                nimp += 1
                        c = cur[k] + nimp
                        if nimp and c < t0 + LDS_LAT:
                            c = t0 + LDS_LAT
                        if big and pipe[k & 3] > c:
                            c = pipe[k & 3]
                        # a new cross-warp import costs an arena slot: weigh it
                        # against start time (IMPORT_PENALTY cycles each)
                        key = (c + IMPORT_PENALTY * nimp, -sum(1 for u in preds[v] if warp_of[u] == k), k)
                        if bt is None or key < bt:
                            bt, w = key, k
                imp = [u for u in preds[v] if warp_of[u] != w and u not in imported[w]]
                if imp and ready < t0 + LDS_LAT:
                    ready = t0 + LDS_LAT
                st = cur[w] + len(imp)
                if big and pipe[w & 3] > st:
                    st = pipe[w & 3]
                if ready > st:
                    st = ready
                if placed and st > limit:
                    deferred.append(v)
                    continue
                imported[w].update(imp)
                cur[w] = st + 1
                if big:
                    pipe[w & 3] = st + cost[v]
                phase_of[v], warp_of[v] = p, w
                finish[v] = st + lat[v]
                if finish[v] > end:
                    end = finish[v]
                order.append(v)
                done.add(v)
                placed += 1
                left -= 1
                for s2 in succs[v]:
                    indeg[s2] -= 1
                    if indeg[s2] == 0:
                        offer(s2)
                bound = lo() + window
                while held and held[0][0] < bound:
                    _, h = heapq.heappop(held)
                    heapq.heappush(heap, (-bl[h], h))
            for v in deferred:
                heapq.heappush(heap, (-bl[v], v))
            t0 = max(end, max(cur)) + BAR
            p += 1
        return t0, phase_of, warp_of, order

    # -- blocks and arena ---------------------------------------------------------
    def _build(self):
        ops = self.em.ops
        self.nphases = 1 + max(self.phase_of.values()) if self.phase_of else 0
        # per warp: [phase] -> [ops] in issue order
        self.blocks = [[[] for _ in range(self.nphases)] for _ in range(self.warps)]
        for v in self.order:
            self.blocks[self.warp_of[v]][self.phase_of[v]].append(v)
        # values read by another warp -> arena slot live from the producing
        # phase to the last phase a consumer on another warp reads it
        last = {}
        for v in self.nodes:
            for r in cg.op_srcs(ops[v]):
                d = self.def_op[r]
                if d in self.warp_of and self.warp_of[d] != self.warp_of[v]:
                    last[r] = max(last.get(r, -1), self.phase_of[v])
        iv = sorted((self.phase_of[self.def_op[r]], b, r) for r, b in last.items())
        self.slot, free, n = {}, [], 0
        for a, b, r in iv:
            if free and free[0][0] < a:  # previous occupant's last read is in an earlier phase
                _, s = heapq.heappop(free)
            else:
                s, n = n, n + 1
            self.slot[r] = s
            heapq.heappush(free, (b, s))
        self.nslots = n

    def critical_path(self):
        """Simulated cycles of one CTA (cost model above)."""
        return self.est

    def total(self):
        return sum(1 for v in self.nodes if self.cost[v])


def split_variants(em, count):
    """Op lists of `count` column variants of a gradient program: every
    variant keeps the ops its own stores need (the prefix, mostly shared)
    plus one contiguous share of the gradient-column tasks; variant 0 also
    stores everything outside the columns (qdd, structural zeros)."""
    tasks = list(dict.fromkeys(t for t in em.tasks if t.startswith("grad.")))
    count = max(1, min(int(count), len(tasks)))
    if count == 1 or not tasks:
        return [em]
    groups = [set(tasks[g * len(tasks) // count:(g + 1) * len(tasks) // count]) for g in range(count)]
    defs = {}
    for i, op in enumerate(em.ops):
        for d in cg.op_dsts(op):
            defs[d] = i
    out = []
    for g, group in enumerate(groups):
        keep = set()
        need = set()
        for i, (op, t) in enumerate(zip(em.ops, em.tasks)):
            if op[0] == "st" and (t in group or (g == 0 and not t.startswith("grad."))):
                keep.add(i)
                need.update(cg.op_srcs(op))
        for i in range(len(em.ops) - 1, -1, -1):
            op = em.ops[i]
            if op[0] != "st" and any(d in need for d in cg.op_dsts(op)):
                keep.add(i)
                need.update(cg.op_srcs(op))
        idx = sorted(keep)
        out.append(cg._sub_emit(em, [em.ops[i] for i in idx], [em.tasks[i] for i in idx]))
    return out


def ptx_warp(sched, w, dtype, scratch_base, out_space, ctab=None, sincos_slots=None):
    """PTX of warp w's whole program: its blocks of every phase, separated by
    `bar.sync 1` (all warps run sched.nphases - 1 barriers).

    Operands: %0 = this lane's input-staging address (shared u32, [slot][33]),
    %1 = this lane's arena address (shared u32, [slot][33]), %2..%4 = out0..2
    (shared u32 [elem][33] when staged, else global u64 per knot), %5 = knot
    valid flag (predicates global stores).  sincos_slots: q slots of the full
    program's sincos ops in order (the rows the prologue fills)."""
    em = sched.em
    ops = em.ops
    t = dtype
    es = 8 if t == "f64" else 4
    R = "%%fd" if t == "f64" else "%%f"
    L = 33
    imm = lambda x: cg._imm(x, t)
    lines = []
    consts = {}
    extra = [em.nreg]
    out_stride = L * es if out_space == "shared" else es
    pred = "@%%p " if out_space == "global" else ""
    # sin/cos scratch rows in the FULL program's order (the kernel prologue
    # fills them; a column variant may use only some joints)
    order = sincos_slots if sincos_slots is not None else [op[3] for op in ops if op[0] == "sincos"]
    at = {sl: k for k, sl in enumerate(order)}
    sc_pos = {}
    for op in ops:
        if op[0] == "sincos":
            sc_pos[op[1]] = scratch_base + 2 * at[op[3]]
            sc_pos[op[2]] = scratch_base + 2 * at[op[3]] + 1
    step = [0]
    have = {}   # reg -> step of its last materialisation in this warp
    mine = set()  # regs computed by this warp's own nodes

    def creg(x):
        if x not in consts:
            consts[x] = extra[0]
            extra[0] += 1
            lines.append(f"mov.{t} {R}{consts[x]}, {imm(x)};")
        return f"{R}{consts[x]}"

    def need(r):
        if r in mine:
            return f"{R}{r}"
        d = sched.def_op[r]
        dop = ops[d]
        if r in have and step[0] - have[r] <= REMAT_DIST:
            return f"{R}{r}"
        if dop[0] == "ld":
            lines.append(f"ld.shared.{t} {R}{r}, [%0+{dop[2] * L * es}];")
        elif dop[0] == "sincos":
            lines.append(f"ld.shared.{t} {R}{r}, [%0+{sc_pos[r] * L * es}];")
        elif em.tasks[d] in REMAT:
            emit(dop, remat=True)
        elif r in sched.slot:
            lines.append(f"ld.shared.{t} {R}{r}, [%1+{sched.slot[r] * L * es}];")
        else:
            raise cg.GenerationError(f"warp {w}: register {r} used before it is available")
        have[r] = step[0]
        return f"{R}{r}"

    def fresh():
        extra[0] += 1
        return f"{R}{extra[0] - 1}"

    def use(a):
        if isinstance(a, float):
            return ctab.operand(a, lines, fresh) if ctab is not None else imm(a)
        return need(a)

    def emit(op, remat=False):
        kd = op[0]
        step[0] += 1
        if kd == "fma":
            a, b, c = op[2], op[3], op[4]
            if isinstance(a, float):
                a, b = b, a
            lines.append(f"fma.rn.{t} {R}{op[1]}, {use(a)}, {use(b)}, {use(c)};")
        elif kd in ("mul", "add"):
            a, b = op[2], op[3]
            if isinstance(a, float):
                a, b = b, a
            lines.append(f"{kd}.rn.{t} {R}{op[1]}, {use(a)}, {use(b)};")
        elif kd == "sub":
            if isinstance(op[2], float):
                lines.append(f"neg.{t} {R}{op[1]}, {use(op[3])};")
                lines.append(f"add.rn.{t} {R}{op[1]}, {R}{op[1]}, {imm(op[2])};")
            else:
                lines.append(f"sub.rn.{t} {R}{op[1]}, {use(op[2])}, {use(op[3])};")
        elif kd == "neg":
            lines.append(f"neg.{t} {R}{op[1]}, {use(op[2])};")
        elif kd == "rcp":
            lines.append(f"rcp.rn.{t} {R}{op[1]}, {use(op[2])};")
        elif kd == "st":
            v = creg(op[3]) if isinstance(op[3], float) else use(op[3])
            lines.append(f"{pred}st.{out_space}.{t} [%{2 + op[1]}+{op[2] * out_stride}], {v};")
            return
        else:
            raise cg.GenerationError(f"unknown op {kd}")
        if remat:
            return
        mine.add(op[1])
        if op[1] in sched.slot:
            lines.append(f"st.shared.{t} [%1+{sched.slot[op[1]] * L * es}], {R}{op[1]};")

    for p in range(sched.nphases):
        if p:
            lines.append("bar.sync 1;")
        for i in sched.blocks[w][p]:
            emit(ops[i])
    head = [f".reg .{t} {R}<{extra[0]}>;"]
    if out_space == "global":
        head += [".reg .pred %%p;", "setp.ne.u32 %%p, %5, 0;"]
    return head + lines
