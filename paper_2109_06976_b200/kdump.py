"""The reference's kernel text format, "rbdkernel v1" (`rbdgen/ir.py:161-227`),
as a wire format in both directions:

* `load_text(text)` parses a dump -- including the reference's own dumps
  under numpy >= 2, whose constants come out as `np.float64(44.145)` and which
  its own `load_text` rejects (`ir.py:180/205`);
* `to_emit(program, dtype)` turns a parsed program (barrier-phased, in-place
  arena slots) into this generator's SSA op list, so the reference's IR for a
  robot can be compiled to an sm_100a kernel (`compile_program`) and run
  batched -- a second, independent device path to diff against the
  generated kernels phase by phase;
* `dump_text(model, alg)` writes this generator's program in the same format
  (one phase per warp-specialised schedule level, one item per task), so the
  two programs can be compared side by side.

IR semantics restated from `ir.py:1-24`: the arena starts zero-filled, inputs
are copied into their segments, phases run in order, items within a phase are
independent, each instruction reads and writes arena slots.
"""

import hashlib
import os
import re
import subprocess

from . import codegen, kernels

FORMAT = "rbdkernel v1"
_OPS = {"fma": 5, "mul": 4, "add": 4, "sub": 4, "neg": 3, "load_const": 3, "sin": 3, "cos": 3, "recip": 3,
        "select": 5}
_FLOAT = re.compile(r"^(?:np\.float64\()?([-+0-9.eEinfa]+)\)?$")


_FOLD = {"fma": lambda a, b, c: a * b + c, "mul": lambda a, b: a * b, "add": lambda a, b: a + b,
         "sub": lambda a, b: a - b, "neg": lambda a: -a, "rcp": lambda a: 1.0 / a}


class KernelFormatError(ValueError):
    """Malformed dump (the reference raises ProgramValidationError, ir.py:75)."""


class Program:
    def __init__(self, arena, inputs, outputs, phases, meta):
        self.arena_size, self.input_map, self.output_map = arena, inputs, outputs
        self.phases, self.meta = phases, meta  # phases: [(label, [item: [(op, dst, args...)]])]


def _const(tok):
    m = _FLOAT.match(tok)
    if not m:
        raise KernelFormatError(f"bad constant {tok!r}")
    return float(m.group(1))


def load_text(text):
    lines = text.splitlines()
    if not lines or not lines[0].startswith("rbdkernel v"):
        raise KernelFormatError("not a kernel dump")
    if lines[0].strip() != FORMAT:
        raise KernelFormatError(f"unsupported kernel format {lines[0].strip()!r}")
    meta, inputs, outputs, phases, item, arena = {}, {}, {}, [], None, 0
    for ln in lines[1:]:
        if not ln.strip():
            continue
        parts = ln.split()
        if ln.startswith("  "):
            op = parts[0]
            if op not in _OPS:
                raise KernelFormatError(f"unknown op {op!r}")
            if item is None:
                raise KernelFormatError("instruction outside an item")
            if op == "load_const":
                item.append((op, int(parts[1]), _const(parts[2])))
            else:
                args = tuple(int(x) for x in parts[1:])
                if len(args) != _OPS[op] - 1:
                    raise KernelFormatError(f"bad arity: {ln!r}")
                item.append((op,) + args)
        elif parts[0] == "meta":
            for kv in parts[1:]:
                k, v = kv.split("=", 1)
                meta[k] = v
        elif parts[0] == "arena":
            arena = int(parts[1])
        elif parts[0] == "input":
            inputs[parts[1]] = (int(parts[2]), int(parts[3]))
        elif parts[0] == "output":
            outputs[parts[1]] = (int(parts[2]), int(parts[3]))
        elif parts[0] == "phase":
            phases.append((parts[1], []))
        elif parts[0] == "item":
            if not phases:
                raise KernelFormatError("item outside a phase")
            item = []
            phases[-1][1].append(item)
        else:
            raise KernelFormatError(f"bad dump line: {ln!r}")
    prog = Program(arena, inputs, outputs, phases, meta)
    validate_program(prog)
    return prog


def validate_program(prog):
    """Structural checks of a parsed dump, restating the reference's
    `validate_program` (ir.py:79-99): a non-empty phase list, every input /
    output segment inside the arena, every instruction slot (destination and
    sources; a load_const's immediate excepted) in [0, arena_size).  A
    truncated or corrupted dump raises here instead of compiling into a
    kernel that silently reads zeros."""
    if not prog.phases:
        raise KernelFormatError("program has no phases")
    size = prog.arena_size
    for name, (off, ext) in list(prog.input_map.items()) + list(prog.output_map.items()):
        if not (0 <= off and off + ext <= size):
            raise KernelFormatError(f"segment {name!r} outside arena")
    for pi, (_, items) in enumerate(prog.phases):
        for wi, item in enumerate(items):
            for ins in item:
                slots = ins[1:2] if ins[0] == "load_const" else ins[1:]
                for sl in slots:
                    if not (0 <= sl < size):
                        raise KernelFormatError(f"phase {pi} item {wi}: slot {sl} outside arena of {size}")


def to_emit(prog, dtype="f64"):
    """SSA op list (`codegen._Emit`) computing the program for one knot.
    Inputs become row loads (q, qd, u order of the algorithm), sin/cos of a
    q slot become the generator's sincos op, outputs become stores in
    output_map order."""
    alg = prog.meta.get("algorithm")
    if alg not in codegen.ALGORITHMS:
        raise KernelFormatError(f"meta algorithm {alg!r} is not one of {codegen.ALGORITHMS}")
    names = list(codegen.INPUTS[alg])
    if set(prog.input_map) != set(names):
        raise KernelFormatError(f"inputs {sorted(prog.input_map)} do not match {alg}")
    n = int(prog.meta.get("n_dof", prog.input_map[names[0]][1]))
    em = codegen._Emit(dtype)
    em.lo, em.np = 0, n
    em.in_layout, off = [], 0
    for nm in names:
        em.in_layout.append((nm, off, n, 0, n))
        off += n
    em.in_total = off
    em.task = "in"
    val = {}  # arena slot -> register id or float
    qslot = {}
    for a, nm in enumerate(names):
        o, e = prog.input_map[nm]
        for i in range(e):
            val[o + i] = em.op("ld", a * n + i)
            if nm == "q":
                qslot[o + i] = i
    sincos = {}

    def get(slot):
        return val.get(slot, 0.0)  # zero-filled arena

    for label, items in prog.phases:
        for k, item in enumerate(items):
            em.task = f"{label}.{k}"
            for ins in item:
                op, dst = ins[0], ins[1]
                if op == "load_const":
                    val[dst] = float(ins[2])
                elif op in ("sin", "cos"):
                    src = ins[2]
                    if src not in qslot or val.get(src) is None or not isinstance(val[src], int):
                        raise KernelFormatError("sin/cos of a value other than a joint position")
                    j = qslot[src]
                    if j not in sincos:
                        s_, c_ = em.reg(), em.reg()
                        em.ops.append(("sincos", s_, c_, j))
                        em.tasks.append("xf")  # joint transforms: re-materialised by consumers
                        sincos[j] = (s_, c_)
                    val[dst] = sincos[j][0 if op == "sin" else 1]
                elif op == "select":
                    raise KernelFormatError("select is not supported (the reference never emits it)")
                else:
                    kind = {"recip": "rcp"}.get(op, op)
                    args = [get(s) for s in ins[2:]]
                    if all(isinstance(a, float) for a in args):  # fold constant-only instructions
                        val[dst] = _FOLD[kind](*args)
                    else:
                        val[dst] = em.op(kind, *args)
    em.task = "out"
    for k, (nm, e) in enumerate(codegen.outputs(alg, n)):
        if nm not in prog.output_map:
            raise KernelFormatError(f"output {nm} missing")
        o, ext = prog.output_map[nm]
        if ext != e:
            raise KernelFormatError(f"output {nm} has extent {ext}, expected {e}")
        for i in range(e):
            v = get(o + i)
            em.store(k, i, v if isinstance(v, float) else codegen.Var(v))
    return em


def dump_text(model, alg, dtype="f64", warps=8):
    """This generator's program for (model, alg) in rbdkernel v1: inputs and
    outputs at the reference's arena offsets, one phase per level of the
    warp-specialised schedule, one item per task; every value its own slot."""
    from . import wsched
    P = wsched.plan(model, alg, dtype, warps)
    em, S = P["em"], P["sched"]
    n = model.n_dof
    slot, nxt = {}, 0
    lines = [FORMAT, f"meta algorithm={alg} generator=paper_2109_06976_b200 model={model.name} n_dof={n}"]
    io = []
    for nm in codegen.INPUTS[alg]:
        io.append(f"input {nm} {nxt} {n}")
        nxt += n
    outs = []
    for nm, e in codegen.outputs(alg, n):
        outs.append((nm, nxt, e))
        io.append(f"output {nm} {nxt} {e}")
        nxt += e
    body = []
    zero = None

    def s_of(a):
        nonlocal nxt, zero
        if isinstance(a, float):
            body.append(f"  load_const {nxt} {float(a)!r}")
            nxt += 1
            return nxt - 1
        return slot[a]

    def emit_op(op):
        nonlocal nxt
        k = op[0]
        if k == "ld":
            slot[op[1]] = op[2]  # inputs sit at their arena offsets
        elif k == "sincos":
            for r, fn in ((op[1], "sin"), (op[2], "cos")):
                slot[r] = nxt
                body.append(f"  {fn} {nxt} {op[3]}")
                nxt += 1
        elif k == "st":
            nm, o, e = outs[op[1]]
            src = s_of(op[3])
            zs = s_of(0.0)
            body.append(f"  add {o + op[2]} {src} {zs}")
        else:
            name = {"rcp": "recip"}.get(k, k)
            args = [s_of(a) for a in op[2:]]
            slot[op[1]] = nxt
            body.append(f"  {name} {nxt} " + " ".join(map(str, args)))
            nxt += 1

    remat = [i for i, t in enumerate(em.tasks) if t in wsched.REMAT]
    body.append("phase setup")
    body.append("item")
    for i in remat:
        emit_op(em.ops[i])
    for p, phase in enumerate(S.phases):
        body.append(f"phase L{p}")
        for tasks in phase:
            for t in tasks:
                body.append("item")
                for i in S.task_ops[t]:
                    emit_op(em.ops[i])
    return "\n".join(lines + [f"arena {nxt}"] + io + body) + "\n"


def compile_program(text, model, dtype="f64", warps=8):
    """Build an sm_100a library running an rbdkernel v1 program batched:
    `rbd_ingested(q, qd, u, out0, out1, out2, N, stream)` (device pointers,
    the layouts of include/rbd_b200.h).  Returns the .so path."""
    prog = load_text(text)
    alg = prog.meta["algorithm"]
    em = to_emit(prog, dtype)
    key = hashlib.sha256((text + dtype + codegen.tuning_key()).encode()).hexdigest()[:16]
    d = os.path.join(kernels.BUILD, f"ingested-{model.name}-{alg}-{dtype}-{key}")
    so = os.path.join(d, "libingested.so")
    if os.path.exists(so):
        return so
    os.makedirs(d, exist_ok=True)
    K = f"Ingested_{alg}_{dtype}"
    # the reference's programs keep every column's partials live at once (its
    # arena), far beyond a thread's registers + row: run them the way they
    # were written -- items of a phase on separate warps, a barrier between
    # phases, cross-item values in the arena (warp-specialised mapping)
    text_k, _, _ = codegen._ws_struct(model, alg, dtype, warps, K, em=em)
    src = "\n".join([
        text_k.replace("#pragma once\n", ""),
        'extern "C" int rbd_ingested(const void* q, const void* qd, const void* u, void* o0, void* o1, void* o2,',
        "                            int64_t N, void* stream) {",
        f"  return rbd_launch_kernel<{K}>(q, qd, u, nullptr, o0, o1, o2, N, stream);",
        "}",
        "",
    ])
    cu = os.path.join(d, "ingested.cu")
    with open(cu, "w") as fh:
        fh.write(src)
    r = subprocess.run([kernels._nvcc()] + kernels.NVCC_FLAGS + ["-shared", "-o", so + ".tmp", cu],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise kernels.BuildError(r.stderr[-4000:])
    os.replace(so + ".tmp", so)
    return so
