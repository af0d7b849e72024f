"""TEST-ONLY: interpreter for the straight-line PTX the generator emits.

Executes the exact text of the inline-asm blocks (codegen.ptx_body for the
thread-per-knot mapping, wsched.ptx_block per phase and warp for the
warp-specialised one) for one knot at a time, with each block's registers
starting empty -- a value a block forgets to load or re-materialise is a
KeyError here, exactly the class of bug the PTX scoping would turn into
garbage on the GPU.  Memory operands are addressed as [%k+offset]; each
operand k maps to a region with its own element stride.
"""
import math
import re

import numpy as np

_MEM = re.compile(r"^(@%p )?(ld|st)\.(shared::cluster|shared|global)\.(f64|f32) (.*)$")
_ADDR = re.compile(r"\[%(\d+)\+(\d+)\]")
_CONST = re.compile(r"^ld\.const\.f64 (\S+), \[(\w+)\+(\d+)\]$")


def _val(tok, regs, f32):
    tok = tok.strip()
    if tok.startswith("0d"):
        return np.frombuffer(bytes.fromhex(tok[2:]), dtype=">f8")[0].item()
    if tok.startswith("0f"):
        return float(np.frombuffer(bytes.fromhex(tok[2:]), dtype=">f4")[0])
    return regs[tok]


def run_block(lines, regions, strides, valid=1, f32=False, consts=None, regs=None):
    """lines: PTX lines (with '%%' escapes as emitted); regions[k]: dict or
    array indexed by element; strides[k]: bytes per element step of operand k.
    regs: register file to continue from (a warp's block split at barriers)."""
    rnd = (lambda x: float(np.float32(x))) if f32 else (lambda x: x)
    regs = {} if regs is None else regs
    for raw in lines:
        ln = raw.replace("%%", "%").strip().rstrip(";")
        if not ln or ln.startswith(".reg") or ln.startswith("setp") or ln.startswith("bar.sync"):
            continue
        if ln.startswith("tcgen05."):  # tensor memory: one lane (this thread), columns by offset
            if ".wait::" in ln:
                continue
            a = re.search(r"\[%(\d+)\+(\d+)\]", ln)
            k, off = int(a.group(1)), int(a.group(2))
            regs_ = re.search(r"\{([^}]*)\}", ln).group(1).split(",")
            first = regs_[0].strip()
            if ln.startswith("tcgen05.st"):
                regions[k][off] = regs[first]
            else:
                for r_ in regs_:
                    regs[r_.strip()] = regions[k][off]
            continue
        if ln.startswith("mov.b64 {") or ln.startswith("mov.b32 %tl"):  # split a value into 32-bit halves
            dst, src = ln.split(" ", 1)[1].rsplit(",", 1)
            for r_ in dst.strip("{} ").split(","):
                regs[r_.strip()] = regs[src.strip()]
            continue
        if ln.startswith("mov.b64 %") and "{" in ln:  # join halves
            dst, src = ln.split(" ", 1)[1].split(",", 1)
            regs[dst.strip()] = regs[src.strip().strip("{}").split(",")[0].strip()]
            continue
        c = _CONST.match(ln)
        if c:
            regs[c.group(1)] = consts[c.group(2)][int(c.group(3)) // 8]
            continue
        m = _MEM.match(ln)
        if m:
            pred, kind, _, _, rest = m.groups()
            if pred and not valid:
                continue
            if kind == "ld":
                dst, addr = [x.strip() for x in rest.split(",", 1)]
                a = _ADDR.search(addr)
                k, off = int(a.group(1)), int(a.group(2))
                regs[dst] = regions[k][off // strides[k]]
            else:
                addr, src = [x.strip() for x in rest.split(",", 1)]
                a = _ADDR.search(addr)
                k, off = int(a.group(1)), int(a.group(2))
                regions[k][off // strides[k]] = _val(src, regs, f32)
            continue
        op, args = ln.split(" ", 1)
        args = [x.strip() for x in args.split(",")]
        d = args[0]
        v = [_val(x, regs, f32) for x in args[1:]]
        base = op.split(".")[0]
        if base == "fma":
            r = v[0] * v[1] + v[2]  # unfused; tolerance-level difference only
        elif base == "mul":
            r = v[0] * v[1]
        elif base == "add":
            r = v[0] + v[1]
        elif base == "sub":
            r = v[0] - v[1]
        elif base == "neg":
            r = -v[0]
        elif base == "rcp":
            r = 1.0 / v[0]
        elif base == "mov":
            r = v[0]
        else:
            raise ValueError(f"unknown PTX op {op}")
        regs[d] = rnd(r)
    return regs


def split_barriers(lines):
    """A warp's block (fsched.ptx_warp) cut at its `bar.sync 1` lines."""
    parts = [[]]
    for ln in lines:
        if ln.strip() == "bar.sync 1;":
            parts.append([])
        else:
            parts[-1].append(ln)
    return parts
