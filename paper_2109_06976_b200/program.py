"""Operator API: the reference's `codegen.build` + `interp.interpret`
(`rbdgen/codegen.py:849-856`, `rbdgen/interp.py:54-86`) on the B200 kernels.

    prog, sched, layout = build(model, "gradFD")
    out = interpret(prog, {"q": q, "qd": qd, "tau": tau})   # {"dq_out": ..., ...}

`build` compiles (or loads) the robot's generated sm_100a library and returns
a `CudaProgram` carrying the reference program's `input_map` / `output_map`
names and extents and its `meta`; `interpret` validates the inputs exactly as
the reference does (`InterpreterError` on a name-set or extent mismatch) and
evaluates them on the GPU.  Inputs may also carry a leading batch axis
(N, extent); outputs then come back as (N, extent).
"""

from dataclasses import dataclass, field

import numpy as np

from . import codegen, kernels, runtime
from .schedule import build_levels
from .urdf import classify_topology


class InterpreterError(ValueError):
    """reference `interp.py:18`"""


@dataclass
class KernelLayout:
    """What replaces the reference's WorkspaceLayout: the batch kernel's
    per-CTA shared-memory staging (one knot per thread)."""
    model_name: str
    algorithm: str
    knots_per_block: int
    smem_bytes_f64: int
    smem_bytes_f32: int
    budget: int | None = None


@dataclass
class CudaProgram:
    model: object
    algorithm: str
    input_map: dict
    output_map: dict
    meta: dict = field(default_factory=dict)
    flops: dict = field(default_factory=dict)

    @property
    def n_dof(self):
        return self.model.n_dof


def build(model, algorithm, budget=None):
    """(CudaProgram, LevelSchedule, KernelLayout) for one robot/algorithm
    (reference `codegen.py:849`)."""
    if algorithm not in codegen.ALGORITHMS:
        raise codegen.GenerationError(f"unsupported algorithm {algorithm!r}")
    lib = kernels.library(model)
    n = model.n_dof
    ins = {nm: (k * n, n) for k, nm in enumerate(codegen.INPUTS[algorithm])}
    outs, off = {}, 0
    for nm, e in codegen.outputs(algorithm, n):
        outs[nm] = (off, e)
        off += e
    meta = {"model": model.name, "algorithm": algorithm, "n_dof": str(n),
            "n_frames": str(model.n_frames), "fused_cross": "0",
            "topology": classify_topology(model), "target": "sm_100a"}
    try:
        fl = kernels.build_meta(model)["flops_per_knot"]
        flops = {d: fl.get(f"{algorithm}_{d}") for d in codegen.DTYPES}
    except OSError:
        flops = {}
    bk = codegen.knots_per_block(model, algorithm, "f64")

    def smem(dt):
        """Shared memory per CTA of the large-batch thread-per-knot kernel
        (knot rows incl. the register plan's parked values); None when the
        robot's large batches run as per-tree parts / split programs."""
        if codegen.tuning(model, algorithm, dt).get("parts"):
            return None
        try:
            L = codegen._layout(model, algorithm, dt, codegen.generate_knot(model, algorithm, dt))
        except codegen.GenerationError:
            return None
        return L["bk"] * L["sin"] * (8 if dt == "f64" else 4)

    layout = KernelLayout(model.name, algorithm, bk, smem("f64"), smem("f32"), budget)
    prog = CudaProgram(model, algorithm, ins, outs, meta, flops)
    prog._lib = lib
    return prog, build_levels(model), layout


def interpret(program, inputs, thread_count=1, dtype="f64"):
    """Run the program on one knot (or a batch); returns {output name: array}
    (reference `interp.py:54-86`).  thread_count is accepted for API parity
    (the GPU decides its own parallelism)."""
    if thread_count < 1:
        raise InterpreterError("thread_count must be positive")
    expected = set(program.input_map)
    got = set(inputs)
    if got != expected:
        raise InterpreterError(f"inputs {sorted(got)} do not match program inputs {sorted(expected)}")
    ndt = np.float64 if dtype == "f64" else np.float32
    arrs, N, single = [], None, None
    for nm in codegen.INPUTS[program.algorithm]:
        _, ext = program.input_map[nm]
        a = np.asarray(inputs[nm], dtype=ndt)
        if a.ndim <= 1:
            a = a.ravel()
            if a.size != ext:
                raise InterpreterError(f"input {nm!r} has {a.size} values, expected {ext}")
            a, s = a.reshape(1, ext), True
        else:
            a = a.reshape(a.shape[0], -1)
            if a.shape[1] != ext:
                raise InterpreterError(f"input {nm!r} has {a.shape[1]} values per knot, expected {ext}")
            s = False
        if N is None:
            N, single = a.shape[0], s
        elif a.shape[0] != N:
            raise InterpreterError("inputs disagree in batch size")
        arrs.append(np.ascontiguousarray(a))
    outs = [np.empty((N, e), dtype=ndt) for _, e in codegen.outputs(program.algorithm, program.n_dof)]
    runtime.run_host(program._lib, program.algorithm, dtype, arrs, outs, N)
    names = [nm for nm, _ in codegen.outputs(program.algorithm, program.n_dof)]
    return {nm: (o[0] if single else o) for nm, o in zip(names, outs)}
