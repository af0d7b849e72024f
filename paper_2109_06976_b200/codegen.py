"""CUDA code generator: one robot -> one sm_100a library of batched kernels.

Replaces the reference's IR generator (`rbdgen/codegen.py:214-856`) and its
Python interpreter (`rbdgen/interp.py`).  Where the reference unrolls the
recursions into a barrier-phased scalar IR executed by a thread pool, this
module unrolls them into ONE straight-line C++ function per (algorithm,
dtype) that evaluates a whole knot point in one CUDA thread:

* every model number (joint axes, origin rotations/translations, inertias,
  gravity) is a literal in the source, so it becomes an FMA immediate /
  constant-bank operand; structural zeros and +-1 factors fold away at
  generation time (`_Emit.lin`), which subsumes the reference's zero-column
  sparsity analysis (`schedule.py:117-139`) -- a gradient column that is
  structurally zero at a frame is simply never emitted;
* independent root trees (fixed base with several limbs: quad12 = 4 legs,
  humanoid30 = torso tree + 2 legs) are emitted one after another; the
  cross-tree blocks of Minv / dID / dFD are literal zeros;
* the mass-matrix inverse is restated column-wise: the articulated-inertia
  factorisation (U, D^-1 per frame) is computed once, then each column of
  Minv is one backward walk up its ancestors and one forward sweep
  (same arithmetic as `refdyn.py:128-169`, reordered so only one 6-vector
  per frame is live);
* gradients are emitted column-major: for each column c (of q and of qd)
  the outward dv/da recursion, the inward df transport and, for gradFD, the
  product -Minv * dc[:, c] are fused, so a column's temporaries die before
  the next column starts (`refdyn.py:178-249` computes all columns at once).

The batch kernel around the per-knot function (input/output staging through
shared memory, coalesced global traffic, launch, host-buffer pipeline) lives
in `csrc/rbd_runtime.cuh`; the C ABI is `include/rbd_b200.h`.
"""

import hashlib
import heapq
import json
import os
import struct

import numpy as np

from . import spatial

ALGORITHMS = ("ID", "Minv", "FD", "gradID", "gradFD")
DTYPES = ("f32", "f64")

# reference operator I/O names (rbdgen/schedule.py:208-226)
INPUTS = {
    "ID": ("q", "qd", "qdd"),
    "Minv": ("q",),
    "FD": ("q", "qd", "tau"),
    "gradID": ("q", "qd", "qdd"),
    "gradFD": ("q", "qd", "tau"),
}


# algorithms whose reference entry takes f_ext (refdyn.py:91-249; minv_direct has none)
FEXT_ALGORITHMS = ("ID", "FD", "gradID", "gradFD")


def input_names(alg, fext=False):
    """Per-knot inputs of a program: the reference operator inputs, plus the
    per-link external forces f_ext [n][6] (link coordinates, refdyn.py:79-80)."""
    if fext and alg not in FEXT_ALGORITHMS:
        raise GenerationError(f"{alg} takes no f_ext")
    return INPUTS[alg] + (("f_ext",) if fext else ())


def input_width(name):
    """Scalars per dof of an input (q, qd, qdd/tau: 1; f_ext: 6)."""
    return 6 if name == "f_ext" else 1


def outputs(alg, n):
    """[(name, extent)] in output_map order."""
    return {
        "ID": [("tau_out", n)],
        "Minv": [("minv_out", n * n)],
        "FD": [("qdd_out", n)],
        "gradID": [("dq_out", n * n), ("dqd_out", n * n)],
        "gradFD": [("dq_out", n * n), ("dqd_out", n * n), ("qdd_out", n)],
    }[alg]


class GenerationError(ValueError):
    """Model outside what the generator supports (reference `codegen.py:49`)."""


# ---------------------------------------------------------------------------
# folded scalar expressions
# ---------------------------------------------------------------------------

class Var:
    """Runtime value `scale * reg` (scale folds into the consumer)."""
    __slots__ = ("name", "scale")

    def __init__(self, name, scale=1.0):
        self.name = name  # register id (int)
        self.scale = float(scale)

    def __neg__(self):
        return Var(self.name, -self.scale)


def neg(e):
    if e is None:
        return None
    if isinstance(e, float):
        return -e if e != 0.0 else None
    return -e


class _Emit:
    """Op-list emitter with constant folding (the generator's IR).

    An entry is None (structural zero), a float (generation-time constant)
    or a Var.  `lin` folds constants, drops zero products, merges repeated
    single terms and returns an alias instead of emitting when the result is
    one scaled register.  Ops (operands: register ids or float immediates):

        ("ld", d, slot)            d = in[slot]      (per-knot input row)
        ("sincos", s, c, slot)     s, c = sin/cos(in[slot])
        ("fma", d, a, b, c) ("mul", d, a, b) ("add", d, a, b) ("sub", d, a, b)
        ("neg", d, a) ("rcp", d, a)
        ("st", k, idx, a)          out_k[idx] = a
    """

    def __init__(self, dtype):
        self.dtype = dtype
        self.ops = []
        self.tasks = []  # task tag of every op (warp-specialised mapping)
        self.task = "main"
        self.nreg = 0
        self.flops = 0  # FMA = 2, MUL/ADD/SUB/RCP = 1 (the reference's counting rule)
        self.lo, self.np = 0, 0  # input dof window of the program (set by _Program.run)
        self.in_layout = []      # [(name, row offset, window length, global offset, global stride)]
        self.in_total = 0        # row slots taken by the inputs
        self.fext = False

    def reg(self):
        self.nreg += 1
        return self.nreg - 1

    def op(self, kind, *args):
        d = self.reg()
        self.ops.append((kind, d) + args)
        self.tasks.append(self.task)
        self.flops += {"fma": 2, "mul": 1, "add": 1, "sub": 1, "rcp": 1}.get(kind, 0)
        return d

    def load(self, slot):
        return Var(self.op("ld", slot))

    def sincos(self, slot):
        s, c = self.reg(), self.reg()
        self.ops.append(("sincos", s, c, slot))
        self.tasks.append(self.task)
        return Var(s), Var(c)

    def rcp(self, e):
        return Var(self.op("rcp", self.operand(e)))

    def operand(self, e):
        """Register id or float immediate holding the entry's value."""
        if e is None:
            return 0.0
        if isinstance(e, float):
            return e
        if e.scale == 1.0:
            return e.name
        if e.scale == -1.0:
            return self.op("neg", e.name)
        return self.op("mul", e.name, e.scale)

    def store(self, k, idx, e):
        v = self.operand(e)
        self.ops.append(("st", k, idx, v))
        self.tasks.append(self.task)

    def lin(self, terms, c0=0.0, hint=None):
        const = float(c0)
        singles = {}
        order = []
        prods = []
        for k, x, y in terms:
            if x is None or y is None or k == 0.0:
                continue
            if isinstance(x, float) and isinstance(y, float):
                const += k * x * y
                continue
            if isinstance(x, float):
                x, y = y, x
            if isinstance(y, float):
                if y == 0.0:
                    continue
                c = k * y * x.scale
                if x.name not in singles:
                    singles[x.name] = 0.0
                    order.append(x.name)
                singles[x.name] += c
                continue
            prods.append((k * x.scale * y.scale, x.name, y.name))
        sing = [(nm, singles[nm]) for nm in order if singles[nm] != 0.0]
        if not prods and not sing:
            return const if const != 0.0 else None
        if not prods and len(sing) == 1 and const == 0.0:
            return Var(sing[0][0], sing[0][1])
        acc = const if const != 0.0 else None
        if acc is None:
            # start the sum from a +-1-scaled single: it becomes the first
            # FMA's addend (no separate multiply or final add; a negation
            # folds into the DFMA operand)
            for idx, (nm, c) in enumerate(sing):
                if c in (1.0, -1.0):
                    acc = nm if c == 1.0 else self.op("neg", nm)
                    sing = sing[:idx] + sing[idx + 1:]
                    break
        for nm, c in sing:
            if acc is None:
                acc = self.op("mul", nm, c) if c not in (1.0, -1.0) else (nm if c == 1.0 else self.op("neg", nm))
            elif c == 1.0:
                acc = self.op("add", nm, acc) if isinstance(acc, float) else self.op("add", acc, nm)
            elif c == -1.0:
                acc = self.op("add", self.op("neg", nm), acc) if isinstance(acc, float) else self.op("sub", acc, nm)
            else:
                acc = self.op("fma", nm, c, acc)
        for c, a, b in prods:
            if c == -1.0:
                a = self.op("neg", a)
            elif c != 1.0:
                a = self.op("mul", a, c)
            acc = self.op("mul", a, b) if acc is None else self.op("fma", a, b, acc)
        return Var(acc)

    def vec(self, rows, hint=None):
        return [self.lin(r, hint=hint) for r in rows]


# ---------------------------------------------------------------------------
# term builders on 6-vectors / 6x6 grids of entries
# ---------------------------------------------------------------------------

def _rows(n=6):
    return [[] for _ in range(n)]


def mv_t(M, v, rows=None):
    """rows[r] += sum_c M[r][c] v[c]."""
    rows = rows if rows is not None else _rows(len(M))
    if v is None:
        return rows
    for r in range(len(M)):
        for c in range(len(v)):
            rows[r].append((1.0, M[r][c], v[c]))
    return rows


def mtv_t(M, v, rows=None):
    """rows[r] += sum_c M[c][r] v[c]  (transpose)."""
    rows = rows if rows is not None else _rows(len(M[0]))
    if v is None:
        return rows
    for r in range(len(M[0])):
        for c in range(len(v)):
            rows[r].append((1.0, M[c][r], v[c]))
    return rows


def add_t(rows, v, k=1.0):
    if v is None:
        return rows
    for r in range(len(rows)):
        rows[r].append((k, v[r], 1.0))
    return rows


def _cross3(rows, off, a, b, k=1.0):
    """rows[off:off+3] += k * (a x b)."""
    rows[off + 0] += [(k, a[1], b[2]), (-k, a[2], b[1])]
    rows[off + 1] += [(k, a[2], b[0]), (-k, a[0], b[2])]
    rows[off + 2] += [(k, a[0], b[1]), (-k, a[1], b[0])]


def mcross_t(v, m, rows=None):
    """rows += v x m = [w x mw; w x ml + l x mw]   (crm, reference spatial.py:45)."""
    rows = rows if rows is not None else _rows()
    if v is None or m is None:
        return rows
    w, l = v[:3], v[3:]
    _cross3(rows, 0, w, m[:3])
    _cross3(rows, 3, w, m[3:])
    _cross3(rows, 3, l, m[:3])
    return rows


def fcross_t(v, f, rows=None):
    """rows += v x* f = [w x fn + l x fg; w x fg]   (crf = -crm^T, spatial.py:68)."""
    rows = rows if rows is not None else _rows()
    if v is None or f is None:
        return rows
    w, l = v[:3], v[3:]
    _cross3(rows, 0, w, f[:3])
    _cross3(rows, 0, l, f[3:])
    _cross3(rows, 3, w, f[3:])
    return rows


def _const_vec(x):
    return [float(t) if float(t) != 0.0 else None for t in x]


def _const_mat(M):
    return [[float(t) if float(t) != 0.0 else None for t in row] for row in M]


def _is_zero_vec(v):
    return v is None or all(e is None for e in v)


# ---------------------------------------------------------------------------
# per-robot program emission
# ---------------------------------------------------------------------------

class _Program:
    def __init__(self, model, alg, dtype):
        self.model = model
        self.alg = alg
        self.em = _Emit(dtype)
        self.n = model.n_dof
        self.parent = list(model.parent)
        self.S = [_const_vec(spatial.motion_subspace(j.kind, j.axis)) for j in model.joints]
        self.I = [_const_mat(ine.spatial()) for ine in model.inertias]
        g = np.asarray(model.gravity, dtype=float)
        self.a0 = _const_vec([0.0, 0.0, 0.0, -g[0], -g[1], -g[2]])
        self.trees = []
        for r in model.roots():
            self.trees.append(model.subtree(r))
        self.E = [None] * self.n
        self.r = [None] * self.n

    # -- inputs and joint transforms -------------------------------------------
    def load_inputs(self, names):
        """Per-knot input row: the program's dof window [lo, lo + np) of each
        input, q at slots [0, np), qd at [np, 2np), u at [2np, 3np), then
        f_ext (6 per dof) when present."""
        em = self.em
        lo, np_, n = em.lo, em.np, self.n
        self.inp = {}
        off = 0
        em.in_layout = []
        for nm in names:
            w = input_width(nm)
            em.in_layout.append((nm, off, w * np_, w * lo, w * n))
            if w == 1:
                self.inp[nm] = [em.load(off + i - lo) if lo <= i < lo + np_ else None for i in range(n)]
            else:
                self.inp[nm] = [[em.load(off + w * (i - lo) + k) for k in range(w)] if lo <= i < lo + np_ else None
                                for i in range(n)]
            off += w * np_
        em.in_total = off

    def emit_xform(self, i):
        """X_i = [[E, 0], [-E skew(r), E]] as an entry grid (folded)."""
        em = self.em
        j = self.model.joints[i]
        E0 = np.asarray(j.origin_rotation, dtype=float).T
        q = self.inp["q"][i]
        if j.kind == "revolute":
            K = spatial.skew(j.axis)
            A = (np.eye(3) + K @ K) @ E0
            B = K @ E0
            C = K @ K @ E0
            sv, cv = em.sincos(i - em.lo)  # q_i sits in input slot i - lo
            E = [[em.lin([(-float(B[r, k]), sv, 1.0), (-float(C[r, k]), cv, 1.0)],
                         c0=float(A[r, k]), hint="e") for k in range(3)] for r in range(3)]
            rv = _const_vec(j.origin_translation)
        elif j.kind == "prismatic":
            E = _const_mat(E0)
            w = np.asarray(j.origin_rotation, dtype=float) @ np.asarray(j.axis, dtype=float)
            rv = [em.lin([(float(w[k]), q, 1.0)], c0=float(j.origin_translation[k]), hint="r")
                  for k in range(3)]
        else:
            raise GenerationError(f"frame {i}: fixed joints must be fused before generation")
        # X_i = [[E, 0], [-E skew(r), E]] is kept factored as (E, r): the
        # lower-left block is never materialised (xm / xtf apply it as
        # E (l - r x w) and r x (E^T f_l)), so a joint costs registers only
        # for the E entries that are not plain +-sin / +-cos aliases.
        self.E[i] = E
        self.r[i] = rv

    def xm(self, i, v, rows=None):
        """rows += X_i v = [E w; E (l - r x w)]."""
        rows = rows if rows is not None else _rows()
        if v is None:
            return rows
        E, rv = self.E[i], self.r[i]
        w, l = v[:3], v[3:]
        rw = _rows(3)
        _cross3(rw, 0, rv, w, -1.0)
        t = self.em.vec([[(1.0, l[k], 1.0)] + rw[k] for k in range(3)], hint="t")
        for r in range(3):
            for k in range(3):
                rows[r].append((1.0, E[r][k], w[k]))
                rows[3 + r].append((1.0, E[r][k], t[k]))
        return rows

    def xtf(self, i, f, rows=None):
        """rows += X_i^T f = [E^T n + r x (E^T l); E^T l]."""
        rows = rows if rows is not None else _rows()
        if f is None:
            return rows
        E, rv = self.E[i], self.r[i]
        n_, l = f[:3], f[3:]
        g = self.em.vec([[(1.0, E[m][k], l[m]) for m in range(3)] for k in range(3)], hint="g")
        for k in range(3):
            for m in range(3):
                rows[k].append((1.0, E[m][k], n_[m]))
            rows[3 + k].append((1.0, g[k], 1.0))
        _cross3(rows, 0, rv, g)
        return rows

    # -- RNEA (reference refdyn.py:55-88) ----------------------------------------
    def emit_rnea(self, tree, qdd, keep=False, v_in=None):
        """Forward v, a, f then backward f accumulation; returns per-frame dicts.
        qdd: per-frame entry list (None entries = zero acceleration)."""
        em = self.em
        qd = self.inp["qd"]
        v, a, f, Xv, Xa, vJ, Iv = {}, {}, {}, {}, {}, {}, {}
        for i in tree:
            p = self.parent[i]
            vJ[i] = [em.lin([(s, qd[i], 1.0)]) if s is not None else None for s in self.S[i]]
            if v_in is not None:
                v[i], Xv[i] = v_in[0][i], v_in[1][i]
            elif p < 0:
                Xv[i] = None
                v[i] = vJ[i]
            else:
                Xv[i] = em.vec(self.xm(i, v[p]), hint="v")
                v[i] = em.vec(add_t(_rows_from(Xv[i]), vJ[i]), hint="v")
            Xa[i] = em.vec(self.xm(i, self.a0 if p < 0 else a[p]), hint="a")
            rows = _rows_from(Xa[i])
            if qdd is not None and qdd[i] is not None:
                for r in range(6):
                    rows[r].append((1.0, qdd[i], self.S[i][r]))
            if p >= 0:
                mcross_t(v[i], vJ[i], rows)
            a[i] = em.vec(rows, hint="a")
            Iv[i] = em.vec(mv_t(self.I[i], v[i]), hint="iv")
            rows = fcross_t(v[i], Iv[i], mv_t(self.I[i], a[i]))
            if em.fext:
                add_t(rows, self.inp["f_ext"][i], -1.0)  # f_i -= f_ext_i (refdyn.py:79-80)
            f[i] = em.vec(rows, hint="f")
        f_local = dict(f)  # per-link forces before the backward accumulation
        tau = {}
        for i in reversed(tree):
            tau[i] = em.lin([(1.0, f[i][r], self.S[i][r]) for r in range(6)], hint="tau")
            p = self.parent[i]
            if p >= 0:
                f[p] = em.vec(add_t(self.xtf(i, f[i]), f[p]), hint="f")
        return dict(v=v, a=a, f=f, Xv=Xv, Xa=Xa, vJ=vJ, Iv=Iv, tau=tau, f_local=f_local)

    def emit_rnea_delta(self, tree, qdd, R0):
        """RNEA at qdd from the RNEA at qdd = 0 of the same (q, qd) (R0):
        the accelerations differ by da_i = X_i da_p + S_i qdd_i -- gravity and
        the velocity-product terms cancel -- so the link forces are
        f_i = f0_i + I_i da_i before the backward pass, and X_i a_p = X_i a0_p
        + X_i da_p.  Same values as emit_rnea(tree, qdd) (refdyn.py:55-88) up
        to rounding, without re-forming I v, v x* I v and v x vJ."""
        em = self.em
        base = em.task
        da, Xa, f = {}, {}, {}
        for i in tree:
            p = self.parent[i]
            rows = _rows()
            Xda = em.vec(self.xm(i, da[p]), hint="xda") if p >= 0 and p in da else None
            if Xda is not None:
                add_t(rows, Xda)
            if qdd[i] is not None:
                for r in range(6):
                    rows[r].append((1.0, qdd[i], self.S[i][r]))
            da[i] = em.vec(rows, hint="da")
            Xa[i] = em.vec(add_t(_rows_from(R0["Xa"][i]), Xda), hint="a") if Xda is not None else R0["Xa"][i]
            rows = mv_t(self.I[i], da[i])
            add_t(rows, R0["f_local"][i])
            f[i] = em.vec(rows, hint="f")
        tau = {}
        for i in reversed(tree):
            tau[i] = em.lin([(1.0, f[i][r], self.S[i][r]) for r in range(6)], hint="tau")
            p = self.parent[i]
            if p >= 0:
                f[p] = em.vec(add_t(self.xtf(i, f[i]), f[p]), hint="f")
        em.task = base
        return dict(v=R0["v"], a=None, f=f, Xv=R0["Xv"], Xa=Xa, vJ=R0["vJ"], Iv=R0["Iv"], tau=tau)

    # -- direct Minv (reference refdyn.py:128-169, column-wise) ------------------
    def emit_minv(self, tree, t=0, store=False, on_column=None):
        em = self.em
        em.task = f"ia.{t}"
        IA = {i: [row[:] for row in self.I[i]] for i in tree}
        U, Dinv = {}, {}
        for i in reversed(tree):
            S = self.S[i]
            U[i] = em.vec([[(1.0, IA[i][r][k], S[k]) for k in range(6)] for r in range(6)], hint="u")
            D = em.lin([(1.0, U[i][k], S[k]) for k in range(6)], hint="d")
            Dinv[i] = em.rcp(D)
            p = self.parent[i]
            if p < 0:
                continue
            ud = [em.lin([(1.0, U[i][c], Dinv[i])], hint="ud") for c in range(6)]
            Ia = [[None] * 6 for _ in range(6)]
            for r in range(6):
                for c in range(r, 6):
                    Ia[r][c] = em.lin([(1.0, IA[i][r][c], 1.0), (-1.0, U[i][r], ud[c])], hint="ia")
                    Ia[c][r] = Ia[r][c]
            # IA_p += X^T Ia X  (symmetric: upper triangle only), as
            # Y = X^T Ia column by column, then rows of Y X = (X^T Y^T)^T
            Y = [self.em.vec(self.xtf(i, [Ia[r][c] for r in range(6)]), hint="ix") for c in range(6)]
            for r in range(6):
                P = self.xtf(i, [Y[c][r] for c in range(6)])
                for c in range(r, 6):
                    IA[p][r][c] = em.lin(P[c] + [(1.0, IA[p][r][c], 1.0)], hint="ia")
                    IA[p][c][r] = IA[p][r][c]
        # per column j: backward walk up the ancestors, then forward sweep
        M = {}
        for j in tree:
            em.task = f"minv.{t}.{j}"
            mb = {}
            F = None
            i = j
            while i >= 0:
                if i == j:
                    m = Dinv[i]
                else:
                    sf = em.lin([(1.0, F[k], self.S[i][k]) for k in range(6)], hint="sf")
                    m = em.lin([(-1.0, Dinv[i], sf)], hint="mb")
                mb[i] = m
                p = self.parent[i]
                if p < 0:
                    break
                rows = _rows()
                add_t(rows, F)
                for r in range(6):
                    rows[r].append((1.0, U[i][r], m))
                F = em.vec(self.xtf(i, em.vec(rows, hint="fb")), hint="fb")
                i = p
            Ff = {}
            for i in tree:
                if i > j:
                    break
                p = self.parent[i]
                if p < 0:
                    M[(i, j)] = mb.get(i)
                    Ff[i] = [em.lin([(s, M[(i, j)], 1.0)]) if s is not None else None for s in self.S[i]]
                else:
                    tt = em.vec(self.xm(i, Ff[p]), hint="ft")
                    ut = em.lin([(1.0, U[i][k], tt[k]) for k in range(6)], hint="ut")
                    M[(i, j)] = em.lin([(1.0, mb.get(i), 1.0), (-1.0, Dinv[i], ut)], hint="m")
                    Ff[i] = em.vec(add_t([[(s, M[(i, j)], 1.0)] if s is not None else []
                                          for s in self.S[i]], tt), hint="ff")
            if store:
                for i in tree:
                    if i > j:
                        break
                    self.store("o0", i * self.n + j, M[(i, j)])
                    if i != j:
                        self.store("o0", j * self.n + i, M[(i, j)])
            if on_column is not None:
                on_column(j, M)
        return M, U, Dinv

    # -- gradient of ID, column-major (reference refdyn.py:178-239) -------------
    def emit_grad_column(self, tree, kind, col, R):
        """dc[:, col] for kind 'q' or 'qd' given the RNEA state R (at qdd)."""
        em = self.em
        dv, da, df = {}, {}, {}
        for i in tree:
            if i < col:
                continue  # column col is zero at frames numbered below it
            p = self.parent[i]
            rows = self.xm(i, dv.get(p)) if p >= 0 else _rows()
            if i == col:
                seed = mcross_t(R["Xv"][i], self.S[i]) if kind == "q" else \
                    [[(s, 1.0, 1.0)] if s is not None else [] for s in self.S[i]]
                for r in range(6):
                    rows[r] += seed[r]
            if i != col and p not in da:
                continue  # frame outside col's subtree: nothing flows out
            dvi = em.vec(rows, hint="dv")
            rows = self.xm(i, da.get(p)) if p >= 0 else _rows()
            mcross_t(dvi, R["vJ"][i], rows)
            if i == col:
                if kind == "q":
                    mcross_t(R["Xa"][i], self.S[i], rows)
                else:
                    mcross_t(R["v"][i], self.S[i], rows)
            dai = em.vec(rows, hint="da")
            dv[i], da[i] = dvi, dai
            Idv = em.vec(mv_t(self.I[i], dvi), hint="idv")
            rows = mv_t(self.I[i], dai)
            fcross_t(R["v"][i], Idv, rows)
            fcross_t(dvi, R["Iv"][i], rows)
            df[i] = em.vec(rows, hint="df")
        dc = {}
        for i in reversed(tree):
            fi = df.get(i)
            if fi is not None:
                dc[i] = em.lin([(1.0, fi[r], self.S[i][r]) for r in range(6)], hint="dc")
            p = self.parent[i]
            if p < 0:
                continue
            rows = _rows()
            if fi is not None:
                self.xtf(i, fi, rows)
            if kind == "q" and i == col:
                add_t(rows, R["xcf"][i])
            if all(not r for r in rows):
                continue
            add_t(rows, df.get(p))
            df[p] = em.vec(rows, hint="df")
        return dc

    def emit_xcf(self, tree, R):
        """X_i^T (S_i x* f_i): the q-derivative of the inward force transport
        (reference refdyn.py:237)."""
        em = self.em
        R["xcf"] = {}
        for i in tree:
            if self.parent[i] < 0:
                continue
            sf = em.vec(fcross_t(self.S[i], R["f"][i]), hint="sf")
            R["xcf"][i] = em.vec(self.xtf(i, sf), hint="xcf")

    # -- drivers -------------------------------------------------------------------
    def store(self, slot, idx, e):
        self.em.store(int(slot[1]), idx, e)

    def run(self, trees=None, zero_fill=True, cols=None, fext=False, lowmem=False, full_window=False, delta=True):
        """Emit the whole one-knot program.  Every op carries a task tag:
        'in' / 'xf' (input loads, joint transforms: re-materialised by each
        consumer), then per root tree t: rnea0.t, ia.t, minv.t.j, fd.t,
        rnea1.t, grad.t.<q|qd>.c, zeros.  The thread-per-knot mapping ignores
        the tags; the warp-specialised mapping schedules tasks over warps."""
        alg, n, em = self.alg, self.n, self.em
        self.lowmem = bool(lowmem)
        part = [t for t in range(len(self.trees)) if trees is None or t in trees]
        dofs = sorted(i for t in part for i in self.trees[t])
        if not dofs or dofs != list(range(dofs[0], dofs[-1] + 1)):
            raise GenerationError(f"part {trees}: its trees must cover a contiguous dof range")
        # full_window: the whole robot's input row and every joint transform
        # (re-materialised on demand), so programs of different parts share
        # one staged row and one sin/cos table (warp-specialised variants)
        em.lo, em.np = (0, n) if full_window else (dofs[0], len(dofs))
        em.fext = bool(fext)
        em.task = "in"
        self.load_inputs(input_names(alg, fext))
        em.task = "xf"
        for i in range(n):
            if full_window or any(i in self.trees[t] for t in part):
                self.emit_xform(i)
        stored = set()
        for t, tree in enumerate(self.trees):
            if t not in part:
                continue
            if alg == "ID":
                em.task = f"rnea0.{t}"
                R = self.emit_rnea(tree, self.inp["qdd"])
                for i in tree:
                    self.store("o0", i, R["tau"][i])
            elif alg == "Minv":
                M, _, _ = self.emit_minv(tree, t, store=True)
                for i in tree:
                    for j in tree:
                        stored.add(i * n + j)
            elif alg == "FD":
                qdd = self._fd(tree, t)[0]
                for i in tree:
                    self.store("o0", i, qdd[i])
            elif alg == "gradID":
                em.task = f"rnea1.{t}"
                R = self.emit_rnea(tree, self.inp["qdd"])
                self.emit_xcf(tree, R)
                for o, kind in (("o0", "q"), ("o1", "qd")):
                    for c in tree:
                        if cols is not None and c not in cols:
                            continue
                        em.task = f"grad.{t}.{kind}.{c}"
                        dc = self.emit_grad_column(tree, kind, c, R)
                        for i in tree:
                            self.store(o, i * n + c, dc.get(i))
                            stored.add(i * n + c)
            elif alg == "gradFD":
                qdd, M, R0 = self._fd(tree, t)
                if cols is None or tree[0] in cols:
                    for i in tree:
                        self.store("o2", i, qdd[i])
                em.task = f"rnea1.{t}"
                if self.lowmem:
                    R = self.emit_rnea(tree, qdd)  # fewer values live across the Minv/FD phase
                elif delta:
                    R = self.emit_rnea_delta(tree, qdd, R0)
                else:
                    R = self.emit_rnea(tree, qdd, v_in=(R0["v"], R0["Xv"]))
                self.emit_xcf(tree, R)
                for o, kind in (("o0", "q"), ("o1", "qd")):
                    for c in tree:
                        if cols is not None and c not in cols:
                            continue
                        em.task = f"grad.{t}.{kind}.{c}"
                        dc = self.emit_grad_column(tree, kind, c, R)
                        for i in tree:
                            terms = [(-1.0, M[(min(i, k), max(i, k))], dc.get(k)) for k in tree]
                            self.store(o, i * n + c, em.lin(terms, hint="o"))
                            stored.add(i * n + c)
            else:
                raise GenerationError(f"unsupported algorithm {alg!r}")
        if alg in ("Minv", "gradID", "gradFD") and zero_fill:
            # cross-tree blocks are structurally zero
            em.task = "zeros"
            for o in (("o0",) if alg == "Minv" else ("o0", "o1")):
                for idx in range(n * n):
                    if idx not in stored:
                        self.store(o, idx, None)
        return self.em

    def _fd(self, tree, t):
        """qdd = Minv (tau - c(q, qd)) (reference refdyn.py:172-175)."""
        em = self.em
        em.task = f"rnea0.{t}"
        R0 = self.emit_rnea(tree, None)
        if self.lowmem:
            # accumulate qdd column by column as Minv is produced, so Minv
            # entries die right after use (same products, summed in column order)
            tau = self.inp["tau"]
            umc = {i: em.lin([(1.0, tau[i], 1.0), (-1.0, R0["tau"][i], 1.0)], hint="umc") for i in tree}
            acc = {i: None for i in tree}

            def add(i, m, k):
                acc[i] = em.lin([(1.0, acc[i], 1.0), (1.0, m, umc[k])], hint="qdd")

            def on_column(j, M):
                for i in tree:
                    if i > j:
                        break
                    add(i, M[(i, j)], j)
                    if i != j:
                        add(j, M[(i, j)], i)

            M, _, _ = self.emit_minv(tree, t, on_column=on_column)
            return acc, M, R0
        M, _, _ = self.emit_minv(tree, t)
        em.task = f"fd.{t}"
        tau = self.inp["tau"]
        umc = {i: em.lin([(1.0, tau[i], 1.0), (-1.0, R0["tau"][i], 1.0)], hint="umc") for i in tree}
        qdd = {}
        for i in tree:
            qdd[i] = em.lin([(1.0, M[(min(i, k), max(i, k))], umc[k]) for k in tree], hint="qdd")
        return qdd, M, R0


def _rows_from(vec):
    rows = _rows()
    if vec is None:
        return rows
    for r in range(6):
        if vec[r] is not None:
            rows[r].append((1.0, vec[r], 1.0))
    return rows


# ---------------------------------------------------------------------------
# source assembly
# ---------------------------------------------------------------------------

_ALG_ENUM = {"ID": 0, "Minv": 1, "FD": 2, "gradID": 3, "gradFD": 4}


def _odd(x):
    return x if x % 2 == 1 else x + 1


# Generation knobs (part of the build key).  RBD_TUNING='{"bk": 128, ...}'
# overrides them for experiments; per-(robot, alg, dtype) overrides live in
# TUNED once measured.
TUNING_DEFAULT = {
    "maps": ["thread", "ws"],  # kernels compiled; launch picks ws for N <= ws_max_n
    "ws_max_n": 8192,    # batch size up to which the (lower-latency) warp-specialised kernel runs
                         # (measured crossover for chain7: ws 20.6 vs thread 28.8 us at 8192,
                         # thread ahead at 16384)
    "warps": 8,          # ws: warps per CTA (one 32-knot group per CTA)
    "minb": 2,           # ws: min CTAs per SM (caps registers at 64K / (32 W minb))
    "bk": 64,            # thread: knots (threads) per CTA
    "sync_every": 0,     # bar.sync every k PTX arithmetic ops (CTA lockstep -> shared I-cache lines)
    "reload_dist": 0,    # re-load smem-resident inputs when the last load is > k ops old (0: load once)
    "stage_kb": 64,      # stage outputs in smem when BK * outputs fit in this many KiB
    "ra": True,          # thread: generator register allocation, spills parked in the smem row
    "warps_per_sm": 16,  # thread + ra: target occupancy (lowered until the row fits)
    "park": True,        # thread + ra: park outputs in the row, coalesced write-back
    "ra_budget": 0,      # thread + ra: cap on values kept in registers (0: from the register cap)
    "prefetch_dist": 0,  # thread + ra: issue reloads up to this many ops before use (0: at use)
    "prefetch_slack": 0,  # ... with at most this many prefetched values in flight
    "fs_warps": 8,       # fs: warps per CTA of the fine-grained schedule
    "fs_variants": 4,    # fs: column variants of a gradient program (CTA rows)
    "fs_max_n": 0,       # fs: batch size up to which the fine-grained kernel runs (with "fs" in maps)
    "ws_variants": 0,    # ws: CTA-row variants of the program (wsched.variant_programs; 0/1: one)
    "wc_cluster": 1,     # wc: CTAs per thread-block cluster sharing one 32-knot group (DSMEM arena)
    "wc_warps": 8,       # wc: warps per CTA
    "wc_variants": 0,    # wc: CTA-row variants
    "wc_max_n": 0,       # wc: batch size up to which the wc kernel runs (with "wc" in maps)
    "rollout_fused": True,  # rollout.Rollout default: one rbd_rollout launch (else per-step launches)
    "wsplit_groups": 6,  # wsplit: column groups of the big tree (CTA-row variants of kernel B)
    "wsplit_warps": 16,  # wsplit: warps of the prefix kernel A
    "wsplit_max_n": 0,   # wsplit: batch size up to which the split small-batch path runs
    "bulk_out": False,   # thread + tmem_row: outputs staged array-major in shared memory and written
                         # back with TMA bulk stores (cp.async.bulk.global.shared::cta), one per array
    "batch_sincos": True,  # thread, fp64: the joints' sin/cos evaluated side by side
                           # (rbd_sincos_batch) instead of one libdevice sincos per joint:
                           # chain7 gradFD 2^20 1.097 -> 1.081 ms, quad12 444 -> 440 us
    "hot_consts": 0,     # thread, fp64: this many most-used table constants held in registers
    "ws_fast_sincos": False,  # ws / fs: each warp's joint sin/cos by rbd_sincos_batch<1> (fp64)
    "l2_prefetch": 0,    # thread: each CTA bulk-prefetches (TMA) the input slabs of the CTA this many
                         # waves (%nsmid SMs x MINB CTAs) ahead into L2 (0: off)
    # read with .get() (absent = off): "tmem_row" (the knot's row in tensor
    # memory), "trow_zmap" (structural zeros unstaged, element-map write-back),
    # "trow_bk" / "trow_ctas" / "trow_stage" (TMEM-row CTA shape experiments),
    # "split*" (split gradient programs), "parts", "zero_memset", "ra_budget"
}
TUNED = {}
# measured on B200 (N = 2^20): chain7 gradFD fp64 is compute-bound at 6 warps/SM
# either way; per-thread output stores beat parking there (1.35 vs 1.43 ms)
TUNED[("chain7", "gradFD", "f64")] = {"park": False, "bk": 32}
# round 2: the knot's row in tensor memory (4-warp CTAs, 2 per SM, 8 warps),
# outputs staged in shared memory and written back coalesced, reloads issued
# up to 24 ops early: 1.24 -> 1.10 ms at N = 2^20 (ncu r2h: IPC 0.90 -> 1.20,
# DRAM 1.64 -> 1.11 GB per launch for 1.06 GB compulsory); fp32 is slower
# that way (0.56 -> 0.84 ms) and keeps the shared-memory row
TUNED[("chain7", "gradFD", "f64")].update({"tmem_row": True, "prefetch_dist": 24, "prefetch_slack": 3})
# the 64 most used fp64 table constants held in registers (loaded once):
# 2^20 1.085 -> 1.069 ms, bit-identical (8 / 16 / 32 / 128: 1.085 / 1.085 /
# 1.074 / 1.078; quad12 loses its third CTA per SM beyond 32)
TUNED[("chain7", "gradFD", "f64")]["hot_consts"] = 64
# the delta form of the second RNEA keeps rnea0's forces live across Minv/FD:
# fewer ops but more spills in chain7's thread-per-knot kernels (2^20: fp64
# 1.093 -> 1.120 ms, fp32 0.563 -> 0.606 ms); their warp-specialised kernels keep it
for _d in DTYPES:
    TUNED.setdefault(("chain7", "gradFD", _d), {})["thread_delta_rnea"] = False
# 32-knot CTAs: finer-grained CTA turnover (staging / write-back barriers),
# measured 1.35 -> 1.22 ms (fp64) and 0.64 -> 0.60 ms (fp32) at N = 2^20
TUNED.setdefault(("chain7", "gradFD", "f32"), {}).update({"bk": 32})
# the fine-grained schedule ("fs", fsched.py) measured slower than the task
# schedule at every small N for chain7 (gradFD fp64 N=128: 10.7 vs 9.9 us;
# ID: 3.4 vs 2.9 us; profiles/small_n_r2.md), so no robot compiles it by default
for _a in ALGORITHMS:
    for _d in DTYPES:
        # measured on B200: with outputs parked in the row, quad12's
        # thread-per-knot kernel runs at ~80% of HBM bandwidth at N = 2^20
        # (3.4x the warp-specialised one); humanoid30's one-knot program
        # (~600 live values) does not fit a thread
        TUNED[("quad12", _a, _d)] = {"warps": 16, "minb": 1, "ws_max_n": 4096,  # thread ahead from 8192
                                     # host path, small N: the one-CTA kernel stages its outputs and writes
                                     # them coalesced over PCIe (gradFD N=128 fp64: 23 us with I/O) --
                                     # faster than the variants + a device->host copy (40 us)
                                     "zc_variants": False}
        if _a in ("gradID", "gradFD"):
            # small batches: CTA-row variants (per leg x column group) spread a
            # 32-knot group over 8 SMs; measured gradFD N=128 fp64 6.2 -> 4.4 us,
            # fp32 5.1 -> 3.3 us (and slower than one CTA from N=1024)
            TUNED[("quad12", _a, _d)].update({"maps": ["thread", "ws", "wc"], "wc_warps": 16, "wc_variants": 8,
                                              "wc_max_n": 256})
        # thread-per-knot kernel: each CTA bulk-prefetches (TMA) the input slabs
        # of the CTA one wave ahead into L2: 2^20 knots gradFD fp64 557 -> 551
        # us, fp32 344 -> 341, FD fp32 91.5 -> 89.0 (tools/experiments)
        TUNED[("quad12", _a, _d)]["l2_prefetch"] = 1
        if _d == "f32" and _a in ("gradFD", "gradID"):
            # 128-knot CTAs for the smem-row fp32 gradients (a longer
            # coalesced write-back per CTA): gradFD 2^20 325 -> 303 us (with
            # 12 warps/SM), gradID 290 -> 275 us; FD / ID / Minv neutral or slower
            TUNED[("quad12", _a, _d)].update({"bk": 128} if _a == "gradID" else {"bk": 128, "warps_per_sm": 12})
        if _d == "f64" and _a in ("gradFD", "gradID", "Minv"):
            # the knot's row in tensor memory (8 warps x 255 registers), the
            # structural zeros (cross-leg blocks) not staged but supplied by
            # the write-back's element map: gradFD 2^20 550 -> 444 us, gradID
            # 436 -> 422, Minv 205 -> 199 (FD / ID and fp32: slower that way)
            TUNED[("quad12", _a, _d)].update({"tmem_row": True, "trow_zmap": True})
        # humanoid30: small batches on the warp-specialised kernel; large ones
        # per root tree (torso tree, two legs)
        TUNED[("humanoid30", _a, _d)] = {"maps": ["ws"], "warps": 16, "minb": 1, "parts": [[0], [1], [2]],
                                         "ws_max_n": 4096,  # measured: parts ahead from 8192 knots
                                         "zero_memset": True, "split": True,
                                         # measured at N = 2^18: per-column programs win in fp32
                                         # (4.6 -> 4.3 ms), lose in fp64 (7.6 -> 8.4 ms)
                                         "split_by_task": _d == "f32",
                                         # knots per split launch pair (measured: fp64 32768, fp32 24576)
                                         "split_chunk": 32768 if _d == "f64" else 24576,
                                         # column-kernel register budget (fp64: 80 + 12 prefetch beat 107 + 12)
                                         "split_budget": 80 if _d == "f64" else 0}
        if _a in ("gradID", "gradFD"):
            # small batches: 10 CTA-row variants (torso column groups + legs) of
            # 8 warps; measured gradFD N=256 fp64 95 -> 41 us, fp32 63 -> 36 us,
            # N=1024 fp64 98 -> 83 us (slower than one CTA per group from 4096)
            TUNED[("humanoid30", _a, _d)].update({"maps": ["ws", "wc"], "wc_warps": 8, "wc_variants": 10,
                                                  "wc_max_n": 256})
            if _d == "f64":
                # 256 < N <= 1024: the split (prefix kernel of 8 warps, then 6
                # column groups + the legs): N=1024 82.6 -> 66.8 us; slower
                # than the variants below (N=256: 37.7 vs 36.2 us)
                TUNED[("humanoid30", _a, _d)].update({"maps": ["ws", "wc", "wsplit"], "wsplit_max_n": 1024,
                                                      "wsplit_warps": 8})
        # the fused rollout runs the one-CTA warp-specialised program (no
        # CTA-row variants: a step's Euler update needs all of a group's
        # outputs); measured B=128 x 32 steps gradFD fp64: fused 2.80 ms vs
        # per-step launches of the variant kernel 1.16 ms
        TUNED[("humanoid30", _a, _d)]["rollout_fused"] = False
        if _d == "f64":
            # the 128 most re-read split-column imports homed in tensor memory
            # and CTA lockstep every 256 ops: gradFD N=2^18 7.46 -> 7.11 ms
            # (ncu r2d: column kernel long-scoreboard stalls 26.8 -> 11.3 per
            # issue, DRAM 1.32 -> 0.86 GB per 32768 knots; then fetch-bound)
            TUNED[("humanoid30", _a, _d)].update({"split_tmem": 128, "sync_every": 256})
            if _a in ("gradFD", "gradID"):
                # 64 most used table constants in registers: gradFD 2^18
                # 6.86 -> 6.78 ms (128 / 256: 6.80 / 6.79)
                TUNED[("humanoid30", _a, _d)]["hot_consts"] = 64


def tuning(model=None, alg=None, dtype=None):
    t = dict(TUNING_DEFAULT)
    if model is not None:
        t.update(TUNED.get((model.name, alg, dtype), {}))
    env = os.environ.get("RBD_TUNING")
    if env:
        t.update(json.loads(env))
    return t


_GEN_SOURCES = []


def _generator_sources():
    """sha256 of the generator sources (computed once per process)."""
    if _GEN_SOURCES:
        return _GEN_SOURCES[0]
    here = os.path.dirname(os.path.abspath(__file__))
    h = hashlib.sha256()
    for f in ("codegen.py", "wsched.py", "fsched.py", os.path.join("csrc", "rbd_runtime.cuh")):
        with open(os.path.join(here, f), "rb") as fh:
            h.update(fh.read())
    _GEN_SOURCES.append(h.hexdigest())
    return _GEN_SOURCES[0]


_TUNING_KEYS = {}


def tuning_key():
    """Build key: generator sources + tuning knobs (a stale build is never reused)."""
    env = os.environ.get("RBD_TUNING", "")
    key = _TUNING_KEYS.get(env)
    if key is None:
        key = hashlib.sha256((_generator_sources() + json.dumps(TUNING_DEFAULT, sort_keys=True)
                              + repr(sorted(TUNED.items())) + env).encode()).hexdigest()[:8]
        _TUNING_KEYS[env] = key
    return key


def knots_per_block(model, alg, dtype):
    """CTA size (knots per block): one knot per thread."""
    return int(tuning(model, alg, dtype)["bk"])


def stage_outputs(model, alg, dtype, bk):
    n = model.n_dof
    ext = sum(e for _, e in outputs(alg, n))
    es = 8 if dtype == "f64" else 4
    return bk * _odd(ext) * es <= tuning(model, alg, dtype)["stage_kb"] * 1024


def generate_knot(model, alg, dtype, trees=None, zero_fill=True, cols=None, fext=False, lowmem=False,
                  full_window=False, delta=None):
    """The one-knot program as an op list (`_Emit`).  trees: restrict to
    these root trees (a 'part'; its outputs are the trees' blocks);
    zero_fill: also store the structural zeros outside the blocks emitted;
    delta: gradFD's second RNEA as a delta from the first (default: tuning
    "delta_rnea")."""
    if delta is None:
        delta = bool(tuning(model, alg, dtype).get("delta_rnea", True))
    return _Program(model, alg, dtype).run(trees, zero_fill, None if cols is None else frozenset(cols), fext,
                                           lowmem, full_window, delta)


_FLOPS = {"fma": 2, "mul": 1, "add": 1, "sub": 1, "rcp": 1}


def _sub_emit(em, ops, tasks):
    """An _Emit holding a subset of another's ops (same registers, inputs)."""
    sub = _Emit(em.dtype)
    sub.ops, sub.tasks, sub.nreg = ops, tasks, em.nreg
    sub.lo, sub.np, sub.in_layout, sub.in_total, sub.fext = em.lo, em.np, em.in_layout, em.in_total, em.fext
    sub.flops = sum(_FLOPS.get(op[0], 0) for op in ops)
    return sub


def split_columns(em, by_task=False):
    """Cut a gradient program into a prefix (RNEA, articulated-inertia
    factorisation, Minv, FD, RNEA at qdd) and its gradient columns.

    Returns (prefix, columns, nx): `prefix` ends every value the columns
    import with ("xst", slot, reg) -- a store to the knot's export slot in an
    L2-resident scratch -- and `columns` starts with ("imp", reg, slot) for
    each of them; inputs and joint transforms are re-materialised on the
    column side.  nx = number of export slots.

    by_task: `columns` is a list with one program per gradient column task
    (an int k: k programs, each a run of consecutive column tasks);
    the joints' sin/cos are exported too (each column program would otherwise
    evaluate every joint's sincos), and each program keeps only the input
    loads / transform entries its column uses."""
    col = [t.startswith("grad.") for t in em.tasks]
    remat = ("in", "xf")
    defs = {}
    for i, op in enumerate(em.ops):
        for d in op_dsts(op):
            defs[d] = i

    def is_remat(di):
        return em.tasks[di] in remat and not (by_task and em.ops[di][0] == "sincos")

    exports = {}
    for i, op in enumerate(em.ops):
        if not col[i]:
            continue
        for r in op_srcs(op):
            di = defs[r]
            if col[di] or is_remat(di):
                continue
            exports.setdefault(r, len(exports))
    if by_task:
        # remat ops feeding exported-by-remat values (transform entries from sin/cos)
        for i, op in enumerate(em.ops):
            if em.tasks[i] in remat and op[0] != "sincos":
                for r in op_srcs(op):
                    if em.ops[defs[r]][0] == "sincos":
                        exports.setdefault(r, len(exports))
    pops, ptasks = [], []
    for i, op in enumerate(em.ops):
        if col[i]:
            continue
        pops.append(op)
        ptasks.append(em.tasks[i])
        for d in op_dsts(op):
            if d in exports:
                pops.append(("xst", exports[d], d))
                ptasks.append(em.tasks[i])
    imps = [("imp", r, sl) for r, sl in exports.items()]
    if not by_task:
        cops = list(imps)
        ctasks = ["imp"] * len(cops)
        for i, op in enumerate(em.ops):
            if col[i] or em.tasks[i] in remat:
                cops.append(op)
                ctasks.append(em.tasks[i])
        return _sub_emit(em, pops, ptasks), _sub_emit(em, cops, ctasks), len(exports)
    progs = []
    tasks = list(dict.fromkeys(t for t in em.tasks if t.startswith("grad.")))
    ng = len(tasks) if by_task is True else max(1, min(int(by_task), len(tasks)))
    groups = [set(tasks[g * len(tasks) // ng:(g + 1) * len(tasks) // ng]) for g in range(ng)]
    for group in groups:
        idx = [i for i, t in enumerate(em.tasks) if t in group]
        need = {r for i in idx for r in op_srcs(em.ops[i])}
        keep = set()
        for i in range(len(em.ops) - 1, -1, -1):  # remat ops this column uses, transitively
            op = em.ops[i]
            if em.tasks[i] in remat and op[0] != "sincos" and any(d in need for d in op_dsts(op)):
                keep.add(i)
                need |= set(op_srcs(op))
        cops = list(imps) + [em.ops[i] for i in sorted(keep | set(idx))]
        ctasks = ["imp"] * len(imps) + [em.tasks[i] for i in sorted(keep | set(idx))]
        progs.append(_sub_emit(em, cops, ctasks))
    return _sub_emit(em, pops, ptasks), progs, len(exports)


def _lit(x, dtype):
    x = float(x)
    return f"{x:.17e}" if dtype == "f64" else f"{np.float32(x):.9e}f"


def _imm(x, dtype):
    if dtype == "f64":
        return "0d%016X" % struct.unpack(">Q", struct.pack(">d", float(x)))[0]
    return "0f%08X" % struct.unpack(">I", struct.pack(">f", float(x)))[0]


def _f64_needs_table(x):
    """fp64 immediates whose low 32 bits are non-zero cannot be encoded in a
    DFMA/DMUL instruction; ptxas would materialise them with UMOV pairs."""
    return (struct.unpack(">Q", struct.pack(">d", float(x)))[0] & 0xFFFFFFFF) != 0


class ConstTable:
    """Per-kernel __constant__ table of the non-encodable fp64 immediates:
    the PTX loads them with ld.const (ptxas turns runs of them into LDCU.128
    uniform loads) instead of two UMOVs per use."""

    def __init__(self, symbol, dtype):
        self.symbol = symbol
        self.on = dtype == "f64"
        self.index = {}

    def operand(self, x, lines, fresh):
        if not self.on or not _f64_needs_table(x):
            return _imm(x, "f64" if self.on else "f32")
        r = fresh()
        lines.append(f"ld.const.f64 {r}, [{self.symbol}+{8 * self.slot(x)}];")
        return r

    def slot(self, x):
        if x not in self.index:
            self.index[x] = len(self.index)
        return self.index[x]

    def declaration(self):
        if not self.index:
            return []
        vals = sorted(self.index, key=self.index.get)
        body = ", ".join(f"{v:.17e}" for v in vals)
        return [f'__constant__ double {self.symbol}[{len(vals)}] = {{{body}}};']


def _input_of_slot(em, slot):
    """(host array name, index within the knot's full input row) of a row slot."""
    for a, (nm, off, w, goff, _) in enumerate(em.in_layout):
        if off <= slot < off + w:
            return ("iq", "iqd", "iu", "ifx")[a], goff + slot - off
    raise GenerationError(f"slot {slot} is not an input")


def cpp_body(em, n):
    """Host C++ backend (test harness only): one statement per op."""
    lit = lambda a: _lit(a, em.dtype) if isinstance(a, float) else f"r{a}"
    out = []
    for op in em.ops:
        k = op[0]
        if k == "ld":
            arr, idx = _input_of_slot(em, op[2])
            out.append(f"const T r{op[1]} = {arr}[{idx}];")
        elif k == "sincos":
            out.append(f"T r{op[1]}, r{op[2]}; rbd_sincos(iq[{em.lo + op[3]}], &r{op[1]}, &r{op[2]});")
        elif k == "fma":
            out.append(f"const T r{op[1]} = rbd_fma({lit(op[2])}, {lit(op[3])}, {lit(op[4])});")
        elif k in ("mul", "add", "sub"):
            sym = {"mul": "*", "add": "+", "sub": "-"}[k]
            out.append(f"const T r{op[1]} = {lit(op[2])} {sym} {lit(op[3])};")
        elif k == "neg":
            out.append(f"const T r{op[1]} = -{lit(op[2])};")
        elif k == "rcp":
            out.append(f"const T r{op[1]} = {_lit(1.0, em.dtype)} / {lit(op[2])};")
        elif k == "st":
            out.append(f"o{op[1]}[{op[2]}] = {lit(op[3])};")
        else:
            raise GenerationError(f"unknown op {k}")
    return out


def op_srcs(op):
    """Register operands an op reads."""
    k = op[0]
    if k == "st":
        args = op[3:4]
    elif k == "xst":
        args = op[2:3]
    elif k in ("ld", "sincos", "imp"):
        args = ()
    else:
        args = op[2:]
    return [a for a in args if not isinstance(a, float)]


def op_dsts(op):
    k = op[0]
    if k in ("st", "xst"):
        return []
    if k == "sincos":
        return [op[1], op[2]]
    return [op[1]]


class SpillPlan:
    """Register allocation of a straight-line op list under a budget of
    `budget` live values, spilling to a per-thread shared-memory row.

    ptxas alone spills a 200-value program to local memory, which on this
    kernel misses L1 (the CTA's shared memory takes most of the carve-out)
    and goes to L2.  Here the generator does it: walking the ops in order it
    keeps at most `budget` values in registers and, when over, evicts the
    value whose next use is furthest away (Belady), storing it once to a
    slot of the knot's shared row; a use of an evicted value reloads it.
    Inputs and the sin/cos scratch already live in the row (their slots are
    their homes, and are recycled once those values die).  Slots of dead
    values are reused, so the row is as long as the peak number of values
    parked at once.

    Result: before[i] = values to (re)load before op i, after[i] = (value,
    slot) stores after op i, slot[v] = row slot of v, nslots = row length."""

    def __init__(self, em, budget, homes, reserved, park_outputs=False, flushes=(), prefetch=None):
        """flushes: (op index, output k) pairs: before that op the CTA writes
        output k back and its parked slots are recycled.  Values defined by
        ("imp", reg, slot) ops (split columns) live in the global scratch:
        evicting them is free, reloading them reads slot `gslot[reg]`."""
        ops = em.ops
        self.park = park_outputs
        self.gslot = {op[1]: op[2] for op in ops if op[0] == "imp"}
        fl = {}
        for i, k in flushes:
            fl.setdefault(i, []).append(k)
        self.outslot = {}  # (output k, element) -> row slot (park_outputs)
        self.outconst = {}  # (output k, element) -> constant value (park_outputs)
        uses = {}
        for i, op in enumerate(ops):
            for a in op_srcs(op):
                uses.setdefault(a, []).append(i)
        ptr = dict.fromkeys(uses, 0)
        self.slot = dict(homes)          # value -> slot (inputs, sin/cos)
        occupied = {sl for v, sl in homes.items() if v in uses}
        free = sorted(set(range(reserved)) - occupied)  # dead / unused input slots
        top = reserved
        inreg = set()
        self.before = {}
        self.after = {}
        self.reloads = self.stores = 0
        far = 1 << 40
        evicted_at = {}   # value -> op index of its last eviction
        reload_log = []   # (value, op index it is needed at, earliest issue point)

        def next_use(v):
            p = ptr[v]
            return uses[v][p] if p < len(uses[v]) else far

        for i, op in enumerate(ops):
            for k in fl.get(i, ()):
                for key, sl in self.outslot.items():
                    if key[0] == k and sl in occupied:
                        occupied.discard(sl)
                        heapq.heappush(free, sl)
            srcs = op_srcs(op)
            for a in srcs:
                if a not in inreg:
                    if a not in self.slot and a not in self.gslot:
                        raise GenerationError(f"value {a} used before it is defined")
                    self.before.setdefault(i, []).append(a)
                    reload_log.append((a, i, evicted_at.get(a, 0)))
                    self.reloads += 1
                    inreg.add(a)
            if park_outputs and op[0] == "st":
                if isinstance(op[3], float):
                    self.outconst[(op[1], op[2])] = op[3]
                else:
                    sl = heapq.heappop(free) if free else top
                    if sl == top:
                        top += 1
                    occupied.add(sl)
                    self.outslot[(op[1], op[2])] = sl
            for a in srcs:
                ptr[a] += 1
            for a in set(srcs):
                if ptr[a] >= len(uses[a]):
                    inreg.discard(a)
                    sl = self.slot.get(a)
                    if sl is not None and sl in occupied:
                        occupied.discard(sl)
                        heapq.heappush(free, sl)
            if op[0] not in ("ld", "sincos", "imp"):
                for d in op_dsts(op):
                    if d in uses:
                        inreg.add(d)
            while len(inreg) > budget:
                v = max(inreg, key=lambda x: (next_use(x), x in self.slot or x in self.gslot))
                inreg.discard(v)
                evicted_at[v] = i + 1
                if v not in self.slot and v not in self.gslot:
                    sl = heapq.heappop(free) if free else top
                    if sl == top:
                        top += 1
                    occupied.add(sl)
                    self.slot[v] = sl
                    self.after.setdefault(i, []).append((v, sl))
                    self.stores += 1
        self.nslots = top
        if prefetch:
            self._prefetch(reload_log, len(ops), *prefetch)

    def _prefetch(self, reload_log, nops, dist, slack):
        """Issue each reload up to `dist` ops before its use (never before the
        value left its register), keeping at most `slack` prefetched values
        in flight at any op: the plan ran with `budget` registers, the
        kernel has budget + slack, so load latency (L2 for split-column
        imports, shared memory otherwise) overlaps the arithmetic."""
        extra = [0] * (nops + 1)
        self.before = {}
        for a, i, lo in reload_log:
            j = max(lo, i - dist, 0)
            for k in range(i - 1, j - 1, -1):
                if extra[k] >= slack:
                    j = k + 1
                    break
            for k in range(j, i):
                extra[k] += 1
            self.before.setdefault(j, []).append(a)


def row_homes(em, scratch_base):
    """Row slot of every input value and sin/cos value of the op list."""
    homes, k = {}, 0
    for op in em.ops:
        if op[0] == "ld":
            homes[op[1]] = op[2]
        elif op[0] == "sincos":
            homes[op[1]], homes[op[2]] = scratch_base + 2 * k, scratch_base + 2 * k + 1
            k += 1
    return homes


def ptx_body(em, scratch_base, out_space, sync_every=0, reload_dist=0, ctab=None, plan=None, tslot=None,
             trow=False, row_base=0, dense=None, hot_consts=0):
    """Device backend: the op list as PTX for one inline-asm block.

    Operand %0 is the 32-bit shared address of the knot's input row (inputs,
    then the sin/cos scratch the C++ prologue fills); %1..%3 address out0..2
    (32-bit shared when staged, 64-bit global otherwise); %4 is 1 for a real
    knot, 0 for the padding threads of the last CTA (their global stores are
    predicated off).  Straight-line PTX goes to ptxas directly (no NVVM pass
    over 10^4-10^5 statements); ptxas allocates registers and schedules.
    sync_every > 0 inserts CTA barriers so all warps walk the instruction
    stream together; reload_dist > 0 re-loads smem-resident values near their
    uses instead of keeping them live.  With a SpillPlan the row also holds
    the values the plan parks: loads and stores follow the plan exactly.
    tslot: {import register: TMEM slot} -- split-column imports homed in
    tensor memory (operand %6 = this thread's TMEM address: lane quadrant of
    its warp, column base): the block starts by copying them scratch -> TMEM
    (tcgen05.st, 32x32b shape: one TMEM lane per thread, an fp64 = 2
    columns), and their reloads are tcgen05.ld, waited for (tcgen05.wait::ld)
    right before the first op that reads one of them.
    trow: the whole row lives in tensor memory (operand %6; row slot s = TMEM
    columns [2 s, 2 s + 2) for fp64): the block starts by copying the staged
    inputs and sin/cos (smem row slots [0, row_base)) into their TMEM homes and
    a CTA barrier (the output staging aliases the input staging); spills are
    tcgen05.st, reloads tcgen05.ld (a reload of a slot stored since the last
    tcgen05.wait::st waits for the stores first).
    Returns (lines, sincos input slots).
    """
    t = em.dtype
    es = 8 if t == "f64" else 4
    R = "%%fd" if t == "f64" else "%%f"
    imm = lambda x: _imm(x, t)
    nreg = em.nreg
    consts = {}
    lines = []
    pred = "@%%p " if out_space == "global" else ""

    def creg(x):
        nonlocal nreg
        if x not in consts:
            consts[x] = nreg
            nreg += 1
            lines.append(f"mov.{t} {R}{consts[x]}, {imm(x)};")
        return f"{R}{consts[x]}"

    home = {}      # register -> smem byte offset it can be re-loaded from
    loaded = {}    # register -> index of its last load
    step = 0

    def fresh():
        nonlocal nreg
        nreg += 1
        return f"{R}{nreg - 1}"

    # the hot_consts most used table constants stay in registers for the
    # whole program (loaded once) instead of a constant load per use
    hot = {}
    if hot_consts and ctab is not None and ctab.on:
        cnt = {}
        for op in em.ops:
            if op[0] in ("fma", "mul", "add", "sub"):
                for a in op[2:]:
                    if isinstance(a, float) and _f64_needs_table(a):
                        cnt[a] = cnt.get(a, 0) + 1
        for x in sorted(cnt, key=lambda v: -cnt[v])[:int(hot_consts)]:
            hot[x] = f"%%hc{len(hot)}"
            lines.append(f"ld.const.f64 {hot[x]}, [{ctab.symbol}+{8 * ctab.slot(x)}];")

    def use(a):
        if isinstance(a, float):
            if a in hot:
                return hot[a]
            return ctab.operand(a, lines, fresh) if ctab is not None else imm(a)
        if plan is not None:
            return f"{R}{a}"
        if a in home and (a not in loaded or (reload_dist and step - loaded[a] > reload_dist)):
            lines.append(f"ld.shared.{t} {R}{a}, [%0+{home[a]}];")
            loaded[a] = step
        return f"{R}{a}"

    sc = []
    narith = 0
    tslot = tslot or {}
    tw = 2 if es == 8 else 1  # TMEM columns per value
    pending = []               # TMEM loads issued, not yet waited for
    st_pending = set()         # TMEM row slots stored since the last tcgen05.wait::st

    def tst(col, reg):
        """store register `reg` (value id) to TMEM column `col`"""
        if es == 8:
            lines.append(f"mov.b64 {{%%tl{reg}, %%th{reg}}}, {R}{reg};")
            lines.append(f"tcgen05.st.sync.aligned.32x32b.x2.b32 [%6+{col}], {{%%tl{reg}, %%th{reg}}};")
        else:
            lines.append(f"mov.b32 %%tl{reg}, {R}{reg};")
            lines.append(f"tcgen05.st.sync.aligned.32x32b.x1.b32 [%6+{col}], {{%%tl{reg}}};")

    def tld(col, reg):
        if es == 8:
            lines.append(f"tcgen05.ld.sync.aligned.32x32b.x2.b32 {{%%tl{reg}, %%th{reg}}}, [%6+{col}];")
        else:
            lines.append(f"tcgen05.ld.sync.aligned.32x32b.x1.b32 {{%%tl{reg}}}, [%6+{col}];")

    if trow:
        if plan is None:
            raise GenerationError("a TMEM row needs a register plan")
        # home slots [0, row_base): staged inputs and the sin/cos the C++
        # prologue wrote; copied through scratch registers %rt (one per slot)
        for g in range(0, row_base, 16):
            grp = range(g, min(g + 16, row_base))
            for sl in grp:
                lines.append(f"ld.shared.{t} %%rt{sl}, [%0+{sl * es}];")
            for sl in grp:
                if es == 8:
                    lines.append(f"mov.b64 {{%%rl{sl}, %%rh{sl}}}, %%rt{sl};")
                    lines.append(f"tcgen05.st.sync.aligned.32x32b.x2.b32 [%6+{tw * sl}], {{%%rl{sl}, %%rh{sl}}};")
                else:
                    lines.append(f"mov.b32 %%rl{sl}, %%rt{sl};")
                    lines.append(f"tcgen05.st.sync.aligned.32x32b.x1.b32 [%6+{tw * sl}], {{%%rl{sl}}};")
        lines.append("tcgen05.wait::st.sync.aligned;")
        lines.append("bar.sync 1;")  # every thread's inputs are in TMEM: the staging may now take outputs
    if tslot:
        if plan is None:
            raise GenerationError("TMEM-homed imports need a register plan")
        items = sorted(tslot.items(), key=lambda x: x[1])
        for g in range(0, len(items), 16):  # 16 scratch loads in flight, then their TMEM stores
            grp = items[g:g + 16]
            for a, _ in grp:
                lines.append(f"ld.global.{t} {R}{a}, [%5+{plan.gslot[a] * 32 * es}];")
            for a, ts in grp:
                if es == 8:
                    lines.append(f"mov.b64 {{%%tl0, %%th0}}, {R}{a};")
                    lines.append(f"tcgen05.st.sync.aligned.32x32b.x2.b32 [%6+{tw * ts}], {{%%tl0, %%th0}};")
                else:
                    lines.append(f"mov.b32 %%tl0, {R}{a};")
                    lines.append(f"tcgen05.st.sync.aligned.32x32b.x1.b32 [%6+{tw * ts}], {{%%tl0}};")
        lines.append("tcgen05.wait::st.sync.aligned;")

    def flush_pending():
        if pending:
            lines.append("tcgen05.wait::ld.sync.aligned;")
            for a in pending:
                if es == 8:
                    lines.append(f"mov.b64 {R}{a}, {{%%tl{a}, %%th{a}}};")
                else:
                    lines.append(f"mov.b32 {R}{a}, %%tl{a};")
            pending.clear()

    for i, op in enumerate(em.ops):
        k = op[0]
        step += 1
        if plan is not None:
            for a in plan.before.get(i, ()):
                if a in tslot:  # TMEM-homed import
                    if a in pending:
                        continue
                    if es == 8:
                        lines.append(f"tcgen05.ld.sync.aligned.32x32b.x2.b32 {{%%tl{a}, %%th{a}}}, [%6+{tw * tslot[a]}];")
                    else:
                        lines.append(f"tcgen05.ld.sync.aligned.32x32b.x1.b32 {{%%tl{a}}}, [%6+{tw * tslot[a]}];")
                    pending.append(a)
                elif a in plan.gslot:  # split columns: import from the knot's scratch slot (L2)
                    lines.append(f"ld.global.{t} {R}{a}, [%5+{plan.gslot[a] * 32 * es}];")
                elif trow:
                    if a in pending:
                        continue
                    sl = plan.slot[a]
                    if sl in st_pending:
                        lines.append("tcgen05.wait::st.sync.aligned;")
                        st_pending.clear()
                    tld(tw * sl, a)
                    pending.append(a)
                else:
                    lines.append(f"ld.shared.{t} {R}{a}, [%0+{plan.slot[a] * es}];")
            if pending and any(a in pending for a in op_srcs(op)):
                flush_pending()
            if k == "sincos":
                sc.append(op[3])
                continue
            if k in ("ld", "imp"):
                continue
        if k == "ld":
            home[op[1]] = op[2] * es
            if not reload_dist:
                use(op[1])
            continue
        if k == "sincos":
            pos = scratch_base + 2 * len(sc)
            sc.append(op[3])
            home[op[1]] = pos * es
            home[op[2]] = (pos + 1) * es
            if not reload_dist:
                use(op[1]), use(op[2])
            continue
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
        elif k == "xst":
            # export to the knot's scratch slot (L2; [32-knot chunk][slot][lane])
            lines.append(f"st.global.{t} [%5+{op[1] * 32 * es}], {use(op[2])};")
        elif k == "st":
            if plan is not None and plan.park:
                if not isinstance(op[3], float):  # constants come from the output map
                    lines.append(f"st.shared.{t} [%0+{plan.outslot[(op[1], op[2])] * es}], {use(op[3])};")
            elif dense is not None:  # staged densely (element map write-back)
                if (op[1], op[2]) not in dense:
                    continue  # a structural zero: the write-back map supplies it
                v = creg(op[3]) if isinstance(op[3], float) else use(op[3])
                lines.append(f"st.shared.{t} [%1+{dense[(op[1], op[2])] * es}], {v};")
            else:
                v = creg(op[3]) if isinstance(op[3], float) else use(op[3])
                lines.append(f"{pred}st.{out_space}.{t} [%{1 + op[1]}+{op[2] * es}], {v};")
        else:
            raise GenerationError(f"unknown op {k}")
        if plan is not None:
            for v, sl in plan.after.get(i, ()):
                if trow:
                    tst(tw * sl, v)
                    st_pending.add(sl)
                else:
                    lines.append(f"st.shared.{t} [%0+{sl * es}], {R}{v};")
        narith += 1
        if sync_every and narith % sync_every == 0:
            lines.append("bar.sync 1;")
    head = [f".reg .{t} {R}<{nreg}>;"]
    if hot:
        head.append(f".reg .f64 %%hc<{len(hot)}>;")
    if tslot or trow:
        head.append(f".reg .b32 %%tl<{em.nreg}>, %%th<{em.nreg}>;")  # TMEM load staging (32-bit halves)
    if trow:
        head.append(f".reg .{t} %%rt<{max(row_base, 1)}>;")
        head.append(f".reg .b32 %%rl<{max(row_base, 1)}>, %%rh<{max(row_base, 1)}>;")
    if out_space == "global":
        head += [".reg .pred %%p;", "setp.ne.u32 %%p, %4, 0;"]
    return head + lines, sc


_MODEL_HASH = {}


def model_hash(model):
    """sha256 of the model's fingerprint (memoised per model object; the
    fingerprint text is recomputed and compared only when the cached entry's
    object has been collected and its id reused)."""
    ent = _MODEL_HASH.get(id(model))
    if ent is not None and ent[0]() is model:
        return ent[1]
    h = hashlib.sha256(model.fingerprint().encode()).hexdigest()
    try:
        import weakref
        _MODEL_HASH[id(model)] = (weakref.ref(model), h)
    except TypeError:
        pass
    return h


SM_SMEM = 228 * 1024      # shared memory per SM (sm_100)
CTA_SMEM_RESERVED = 1024  # per-CTA system reservation
REG_OVERHEAD = 16         # registers ptxas needs besides the budgeted values


def _layout(model, alg, dt, em, device=True, over=None):
    """Thread-per-knot launch shape and row layout.

    Without the allocator ("ra": false) the row is [inputs | sin/cos] and
    ptxas allocates registers alone.  With it, the generator keeps at most
    B values in registers (B from the per-thread register cap at the target
    warps per SM) and parks the rest in the knot's shared-memory row; the
    target occupancy is lowered until the row fits the SM's shared memory."""
    n = model.n_dof
    outs = outputs(alg, n)
    ext = [e for _, e in outs] + [0] * (3 - len(outs))
    nin = len(em.in_layout)
    nsc = sum(1 for op in em.ops if op[0] == "sincos")
    tn = tuning(model, alg, dt)
    tn.update(over or {})
    bk = int(tn["bk"])
    es = 8 if dt == "f64" else 4
    base = em.in_total + 2 * nsc
    sout = _odd(sum(ext))
    plan, minb = None, 1
    if tn.get("tmem_row") and tn.get("ra") and device:
        # the knot's row (inputs, sin/cos, spilled values) lives in tensor
        # memory, one TMEM lane per thread (2 columns per fp64): 4-warp CTAs,
        # 2 per SM (8 warps, 255 registers), each CTA 256 columns; shared
        # memory only stages the inputs and then, aliased over them, the
        # outputs in element order for the coalesced write-back (with
        # trow_zmap only the non-zero ones: a third CTA then fits the shared
        # memory and waits in tcgen05.alloc with its inputs staged)
        tbk = int(tn.get("trow_bk", 128))  # 256: one 8-warp CTA per SM (all warps on one TMEM allocation)
        # CTAs per SM: 2 (255 registers, 256 TMEM columns per thread); 3-4
        # with per-thread global output stores (no output staging; 170 / 128
        # registers, 128 columns)
        tstage = bool(tn.get("trow_stage", True))
        ctas_sm = int(tn.get("trow_ctas", 256 // tbk))
        tcols_thread = 1 << ((512 // (ctas_sm * (tbk // 128))).bit_length() - 1)
        budget = (min(255, 65536 // (ctas_sm * tbk)) - REG_OVERHEAD) // (2 if dt == "f64" else 1)
        if tn.get("ra_budget"):
            budget = min(budget, int(tn["ra_budget"]))
        pf = None
        if tn.get("prefetch_dist"):
            pf = (int(tn["prefetch_dist"]), int(tn["prefetch_slack"]))
            budget -= pf[1]
        homes = row_homes(em, em.in_total)
        plan = SpillPlan(em, budget, homes, base, park_outputs=False, prefetch=pf)
        tw = 2 if es == 8 else 1
        row = _odd(base)
        smem = tbk * max(row, sout) * es
        # a row longer than a TMEM lane (e.g. the f_ext program), or outputs
        # that do not fit the staging of 2 CTAs, keep the shared-memory row
        # a part program (a subset of the root trees) stages only the elements
        # it stores, densely, and writes them back through an element map
        stored = sorted({(op[1], op[2]) for op in em.ops if op[0] == "st"})
        offs = [0, ext[0], ext[0] + ext[1]]
        tpart = zmap = dense = None
        if len(stored) < sum(ext):
            tpart = [offs[k] + idx for k, idx in stored]
            dense = {kv: j for j, kv in enumerate(stored)}
            sout_t = _odd(len(stored))
        else:
            sout_t = sout
            nonzero = sorted({(op[1], op[2]) for op in em.ops
                              if op[0] == "st" and not (isinstance(op[3], float) and op[3] == 0.0)})
            if tn.get("trow_zmap") and len(nonzero) < sum(ext):
                # structural zeros (e.g. cross-leg blocks) are not staged:
                # the write-back takes element e from dense slot zmap[e], or 0
                dense = {kv: j for j, kv in enumerate(nonzero)}
                zmap = [-1] * sum(ext)
                for (k, idx), j in dense.items():
                    zmap[offs[k] + idx] = j
                sout_t = _odd(len(nonzero))
        if not tstage:
            sout_t, tpart, zmap, dense = 0, None, None, None
        smem = tbk * max(row, sout_t) * es + (2 * len(zmap) if zmap else 0)
        if plan.nslots * tw <= tcols_thread and ctas_sm * (smem + CTA_SMEM_RESERVED) <= SM_SMEM:
            return dict(n=n, ext=ext, nin=nin, nsc=nsc, bk=tbk, stage=tstage, sin=row, sout=sout_t, plan=plan,
                        minb=ctas_sm, park=False, lo=em.lo, np=em.np, in_layout=em.in_layout, trow=True,
                        tcols=tmem_alloc(tcols_thread, tbk),
                        bulk=bool(tstage and tpart is None and zmap is None and tn.get("bulk_out")),
                        tpart=tpart, zmap=zmap, dense=dense)
        plan = None
    if tn.get("ra") and device:
        homes = row_homes(em, em.in_total)
        for warps in range(int(tn["warps_per_sm"]), 1, -1):
            threads = 32 * warps
            if threads % bk:
                continue
            ctas = threads // bk
            regs = min(255, 65536 // threads)
            budget = (regs - REG_OVERHEAD) // (2 if dt == "f64" else 1)
            if tn.get("ra_budget"):
                budget = min(budget, int(tn["ra_budget"]))
            pf = None
            if tn.get("prefetch_dist"):
                pf = (int(tn["prefetch_dist"]), int(tn["prefetch_slack"]))
                budget -= pf[1]
            park = bool(tn.get("park", True))
            row_max = (SM_SMEM - ctas * (CTA_SMEM_RESERVED + (4 * sum(ext) if park else 0) + 16)) // (threads * es)
            plan = SpillPlan(em, budget, homes, base, park_outputs=park, prefetch=pf)
            if _odd(plan.nslots) <= row_max:
                minb = ctas
                break
        else:
            raise GenerationError(f"{model.name} {alg} {dt}: no occupancy fits the spill row")
        row = _odd(max(base, plan.nslots))
        # parked: outputs parked in the row and written back coalesced; else
        # each thread stores its outputs to global as they are produced
        stage = False
        bad = {v for v in plan.outconst.values() if v != 0.0}
        if bad:
            raise GenerationError(f"{model.name} {alg}: constant outputs {bad} other than 0")
    else:
        row = _odd(base)
        stage = stage_outputs(model, alg, dt, bk)
    return dict(n=n, ext=ext, nin=nin, nsc=nsc, bk=bk, stage=stage, sin=row, sout=sout,
                plan=plan, minb=minb, park=plan is not None and plan.park, lo=em.lo, np=em.np,
                in_layout=em.in_layout)


def _input_consts(layout):
    """Per-input staging constants of a kernel struct: window length, offset
    and stride in the knot's global row, offset in the knot's smem row."""
    def fn(name, idx):
        body = " : ".join(f"a == {a} ? {ent[idx]}" for a, ent in enumerate(layout)) + " : 0"
        return f"  RBD_HDC static constexpr int {name}(int a) {{ return {body}; }}"
    return [fn("inw", 2), fn("ing", 3), fn("ins", 4), fn("inr", 1)]


def _struct_head(model, alg, dt, L, fl, name=None):
    T = "double" if dt == "f64" else "float"
    return [
        f"struct {name or f'Knot_{alg}_{dt}'} {{",
        f"  typedef {T} T;",
        f"  static constexpr int NDOF = {L['n']}, NIN = {L['nin']}, BK = {L['bk']};",
        f"  static constexpr int LO = {L['lo']}, NP = {L['np']};  // input dof window [LO, LO + NP)",
    ] + _input_consts(L["in_layout"]) + [
        f"  static constexpr int E0 = {L['ext'][0]}, E1 = {L['ext'][1]}, E2 = {L['ext'][2]};",
        f"  static constexpr int SIN = {L['sin']}, SOUT = {L['sout']};",
        f"  static constexpr bool STAGE = {'true' if L['stage'] else 'false'};",
        f"  static constexpr bool PARK = {'true' if L.get('park') else 'false'};  // outputs parked in the row",
        f"  static constexpr int FLOPS = {fl};",
        "  static constexpr int MAP = 0;  // thread per knot",
        f"  static constexpr int MINB = {L.get('minb', 1)};  // CTAs per SM the row layout is sized for",
        f"  static constexpr int TCOLS = {L.get('tcols', 0)};  // TMEM columns per CTA (split-column imports / row)",
        f"  static constexpr bool TROW = {'true' if L.get('trow') else 'false'};  // the row lives in TMEM; "
        "outputs staged over the input staging",
        f"  static constexpr bool TPART = {'true' if L.get('tpart') else 'false'};  // ... densely, a part's "
        "elements only",
        f"  static constexpr int L2PF = {int(tuning(model, alg, dt).get('l2_prefetch', 0))};  // input slabs "
        "bulk-prefetched into L2 this many CTA waves ahead (0: off)",
        f"  static constexpr bool BULK = {'true' if L.get('bulk') else 'false'};  // outputs staged array-major, "
        "written back by TMA bulk stores",
    ]


def _omap(L):
    """Parked-output list of the program: [(element, slot)] in element order,
    element = index into the outputs concatenated in output_map order, slot
    = row slot holding it or -1 for a structural 0.  A part program (a subset
    of the root trees) lists only the elements it writes."""
    plan = L["plan"]
    out, base = [], 0
    for k, e in enumerate(L["ext"]):
        for idx in range(e):
            if (k, idx) in plan.outslot:
                out.append((base + idx, plan.outslot[(k, idx)]))
            elif (k, idx) in plan.outconst:
                out.append((base + idx, -1))
        base += e
    return out


def _omap_decl(L, name):
    if not L.get("park"):
        return []
    om = _omap(L)
    full = [e for e, _ in om] == list(range(sum(L["ext"])))
    if full is False and L.get("full_outputs"):
        raise GenerationError(f"{name}: some outputs are never written")
    if sum(L["ext"]) > 65535:
        raise GenerationError(f"{name}: output map too large")
    L["nout"], L["ofull"] = len(om), full
    pad = om or [(0, -1)]  # a program with no outputs (split gradID prefix) keeps a 1-entry dummy map
    lines = [f"__constant__ short rbd_om_{name}[{len(pad)}] = {{{', '.join(str(sl) for _, sl in pad)}}};"]
    if not full:
        lines.append(f"__constant__ unsigned short rbd_oe_{name}[{len(pad)}] = "
                     f"{{{', '.join(str(e) for e, _ in pad)}}};")
    return lines


def tmem_homes(plan, count, es):
    """{import register: TMEM slot} for the `count` split-column imports the
    plan reloads most often, and the TMEM columns a CTA allocates for them
    (power of two >= 32; an fp64 takes 2 columns of the thread's lane)."""
    if not count or plan is None or not plan.gslot:
        return {}, 0
    hits = {}
    for lst in plan.before.values():
        for a in lst:
            if a in plan.gslot:
                hits[a] = hits.get(a, 0) + 1
    top = sorted(hits, key=lambda a: (-hits[a], a))[:int(count)]
    cols = (2 if es == 8 else 1) * len(top)
    if cols == 0:
        return {}, 0
    return {a: k for k, a in enumerate(top)}, cols


def tmem_alloc(cols_per_thread, bk):
    """TMEM columns a CTA of bk threads allocates when each thread needs
    cols_per_thread columns of its lane: warps w and w + 4 share lane
    quadrant w % 4 and split the columns (power of two >= 32, <= 512)."""
    per = bk // 128
    alloc = 32
    while alloc < cols_per_thread * per:
        alloc *= 2
    if alloc > 512:
        raise GenerationError(f"{cols_per_thread} TMEM columns x {per} warps per quadrant exceed 512")
    return alloc


def _knot_struct(model, alg, dt, name=None, trees=None, zero_fill=True, fext=False, em=None, nx=0, over=None,
                 tmem=0):
    """Device header: C++ sin/cos prologue + the PTX body in one asm block.
    nx > 0: the program exports nx values per knot to the split scratch;
    tmem > 0: that many of the imports it reloads most are homed in tensor
    memory (tmem_homes) -- the CTA must be 4 warps (one per TMEM lane quadrant)."""
    if em is None:
        tk = tuning(model, alg, dt)
        em = generate_knot(model, alg, dt, trees, zero_fill, fext=fext,
                           delta=bool(tk.get("thread_delta_rnea", tk.get("delta_rnea", True))))
    L = _layout(model, alg, dt, em, over=over)
    n = L["n"]
    space = "shared" if L["stage"] else "global"
    tn = tuning(model, alg, dt)
    ctab = ConstTable(f"rbd_c_{name or f'Knot_{alg}_{dt}'}", dt)
    plan = L["plan"]
    if L.get("trow"):
        tslot = {}
    else:
        tslot, tc = tmem_homes(plan, tmem, 8 if dt == "f64" else 4)
        if tslot and L["bk"] % 128:
            raise GenerationError("TMEM-homed imports need CTAs of 4k warps (warps spread over the TMEM lane "
                                  "quadrants)")
        L["tcols"] = tmem_alloc(tc, L["bk"]) if tslot else 0
    body, sc = ptx_body(em, em.in_total, space, tn["sync_every"], tn["reload_dist"], ctab, plan, tslot=tslot,
                        trow=bool(L.get("trow")), row_base=L["sin"] if L.get("trow") else 0, dense=L.get("dense"),
                        hot_consts=int(tn.get("hot_consts", 0)))
    ra = (f"// register budget: {plan.reloads} reloads, {plan.stores} parked values, row {L['sin']} slots, "
          f"{L['minb']} CTAs of {L['bk']} per SM" if plan is not None else "// ptxas register allocation")
    src = [
        f"// GENERATED by paper_2109_06976_b200.codegen -- robot {model.name!r}, {alg} {dt}",
        f"// {em.flops} flops per knot (FMA = 2, MUL/ADD/SUB/RCP = 1); {em.nreg} SSA registers",
        ra,
        "#pragma once",
        '#include "rbd_runtime.cuh"',
    ] + ctab.declaration() + _omap_decl(L, name or f"Knot_{alg}_{dt}") \
        + _struct_head(model, alg, dt, L, em.flops, name) + [
        f"  static constexpr int NX = {nx};  // values exported per knot to the split scratch",
    ]
    if L.get("tpart"):
        nm = name or f"Knot_{alg}_{dt}"
        src.insert(src.index("#pragma once") + 2,
                   f"__constant__ unsigned short rbd_te_{nm}[{len(L['tpart'])}] = "
                   f"{{{', '.join(str(e) for e in L['tpart'])}}};")
        src.append(f"  static constexpr int NOUT = {len(L['tpart'])};  // output elements this part writes")
        src.append(f"  __device__ __forceinline__ static const unsigned short* oelem() {{ return rbd_te_{nm}; }}")
    if L.get("zmap"):
        nm = name or f"Knot_{alg}_{dt}"
        src.insert(src.index("#pragma once") + 2,
                   f"__constant__ short rbd_zm_{nm}[{len(L['zmap'])}] = "
                   f"{{{', '.join(str(e) for e in L['zmap'])}}};")
        src.append(f"  static constexpr int NZM = {len(L['zmap'])};  // output elements: dense staging slot or -1 (0)")
        src.append(f"  __device__ __forceinline__ static const short* zmap() {{ return rbd_zm_{nm}; }}")
    if L.get("park"):
        nm = name or f"Knot_{alg}_{dt}"
        src.append(f"  static constexpr int NOUT = {L['nout']};  // output elements this program writes")
        src.append(f"  static constexpr bool OFULL = {'true' if L['ofull'] else 'false'};  // ... all of them, in order")
        src.append(f"  __device__ __forceinline__ static const short* omap() {{ return rbd_om_{nm}; }}")
        src.append("  __device__ __forceinline__ static const unsigned short* oelem() { return "
                   + (f"rbd_oe_{nm}" if not L["ofull"] else "nullptr") + "; }")
    src += ["  __device__ __forceinline__ static void run_dev(T* my, T* o0, T* o1, T* o2, unsigned valid, T* xb,",
            "                                                 unsigned tm = 0) {",
            "    (void)tm;"]
    base = em.in_total
    if sc and dt == "f64" and tn.get("batch_sincos"):
        nsc = len(sc)
        src.append(f"    {{ double x_[{nsc}] = {{{', '.join(f'my[{slot}]' for slot in sc)}}}, s_[{nsc}], c_[{nsc}];")
        src.append(f"      rbd_sincos_batch<{nsc}>(x_, s_, c_);")
        for k in range(nsc):
            src.append(f"      my[{base + 2 * k}] = s_[{k}]; my[{base + 2 * k + 1}] = c_[{k}];")
        src.append("    }")
    else:
        for k, slot in enumerate(sc):
            src.append(f"    {{ T s, c; rbd_sincos(my[{slot}], &s, &c); my[{base + 2 * k}] = s; "
                       f"my[{base + 2 * k + 1}] = c; }}")
    src.append("    const unsigned a_in = (unsigned)__cvta_generic_to_shared(my);")
    if L["stage"]:
        src.append("    const unsigned a0 = (unsigned)__cvta_generic_to_shared(o0), "
                   "a1 = (unsigned)__cvta_generic_to_shared(o1), a2 = (unsigned)__cvta_generic_to_shared(o2);")
        ops = '"r"(a_in), "r"(a0), "r"(a1), "r"(a2), "r"(valid), "l"(xb), "r"(tm)'
    else:
        ops = '"r"(a_in), "l"(o0), "l"(o1), "l"(o2), "r"(valid), "l"(xb), "r"(tm)'
    src.append('    asm volatile("{\\n\\t"')
    for ln in body:
        src.append(f'      "{ln}\\n\\t"')
    src.append(f'      "}}" :: {ops} : "memory");')
    src += ["  }", "};", ""]
    return "\n".join(src), em.flops, L


def _multi_knot_struct(model, alg, dt, name, progs, nx, over, tmem=0):
    """One thread-per-knot kernel holding several one-knot programs (the
    gradient columns of a split program); CTA row blockIdx.y runs program
    blockIdx.y, so every warp of a CTA streams the same (short) code.  All
    programs share the register cap and row length of the most demanding."""
    Ls = [_layout(model, alg, dt, p, over=over) for p in progs]
    warps = min(L["minb"] * L["bk"] // 32 for L in Ls)
    over = dict(over, warps_per_sm=warps)
    Ls = [_layout(model, alg, dt, p, over=over) for p in progs]
    L0 = dict(Ls[0])
    L0["sin"] = _odd(max(L["sin"] for L in Ls))
    L0["minb"] = min(L["minb"] for L in Ls)
    flops = sum(p.flops for p in progs)
    head = [
        f"// GENERATED by paper_2109_06976_b200.codegen -- robot {model.name!r}, {alg} {dt}, "
        f"{len(progs)} column programs",
        f"// {flops} flops per knot over all programs; row {L0['sin']} slots, {L0['minb']} CTAs of {L0['bk']} per SM",
        '#include "rbd_runtime.cuh"',
    ]
    bodies, decls = [], []
    tcols = 0
    if tmem and L0["bk"] % 128:
        raise GenerationError("TMEM-homed imports need CTAs of 4k warps")
    for k, (p, L) in enumerate(zip(progs, Ls)):
        ctab = ConstTable(f"rbd_c_{name}_{k}", dt)
        # each program homes ITS most re-read imports in tensor memory
        tslot, tc = tmem_homes(L["plan"], tmem, 8 if dt == "f64" else 4)
        if tslot:
            tcols = max(tcols, tmem_alloc(tc, L0["bk"]))
        body, sc = ptx_body(p, p.in_total, "global", 0, 0, ctab, L["plan"], tslot=tslot)
        if sc:
            raise GenerationError("column programs import their sin/cos")
        decls += ctab.declaration()
        bodies.append((p.tasks[-1], body))
    L0["tcols"] = tcols
    src = head + decls + _struct_head(model, alg, dt, L0, flops, name) + [
        f"  static constexpr int NX = {nx};  // values per knot in the split scratch",
        f"  static constexpr int NPROG = {len(progs)};",
        "  __device__ __forceinline__ static void run_dev(T* my, T* o0, T* o1, T* o2, unsigned valid, T* xb,",
        "                                                 unsigned tm = 0) {",
        "    run_prog(blockIdx.y, my, o0, o1, o2, valid, xb, tm);",
        "  }",
        "  __device__ __forceinline__ static void run_prog(int prog, T* my, T* o0, T* o1, T* o2, unsigned valid,",
        "                                                  T* xb, unsigned tm) {",
        "    (void)tm;",
        "    const unsigned a_in = (unsigned)__cvta_generic_to_shared(my);",
        "    switch (prog) {",
    ]
    for k, (task, body) in enumerate(bodies):
        src.append(f"    case {k}:  // {task}")
        src.append('      asm volatile("{\\n\\t"')
        for ln in body:
            src.append(f'        "{ln}\\n\\t"')
        src.append('        "}" :: "r"(a_in), "l"(o0), "l"(o1), "l"(o2), "r"(valid), "l"(xb), "r"(tm) : "memory");')
        src.append("      break;")
    src += ["    default: break;", "    }", "  }", "};", ""]
    return "\n".join(src)


def _ws_struct(model, alg, dt, warps, name=None, trees=None, zero_fill=True, fext=False, em=None, variants=0,
               cluster=1, progs=None, ext=None):
    """Device header of the warp-specialised mapping (see wsched.py).  With
    an `em` holding "imp" ops (split columns), the arena is the per-group
    slice of the split scratch the prefix kernel filled.  variants > 1: the
    program is cut into CTA-row variants (wsched.variant_programs; blockIdx.y
    picks one), each scheduled on its own; outputs go straight to global.
    cluster > 1: the tasks are scheduled over cluster x warps warps of a
    thread-block cluster (one 32-knot group per cluster, CTA rank r runs warps
    [r W, (r + 1) W)); a task reads a value another CTA produced from that
    CTA's shared-memory arena (DSMEM, ld.shared::cluster) and phases end with
    a cluster barrier -- each SM streams only its own warps' code."""
    from . import wsched
    C = max(1, int(cluster))
    sw = warps * C  # warps the tasks are scheduled over
    if progs is not None:
        pass  # explicit variant programs (wsched.split_programs)
    elif variants and variants > 1 and em is None and trees is None:
        progs = wsched.variant_programs(model, alg, dt, variants, fext)
    if progs is not None and len(progs) > 1:
        Ps = [wsched.plan(model, alg, dt, sw, em=e, ext=ext) for e in progs]
        P = dict(Ps[0])
        na = max(p["sched"].nslots for p in Ps)
        row = wsched.LANES * P["es"]
        P["arena_smem"] = row * (P["sin"] + na) <= wsched.SMEM_BUDGET
        P["stage"] = False
    else:
        P = wsched.plan(model, alg, dt, sw, trees, zero_fill, fext, em=em, ext=ext)
        Ps = [P]
        na = P["sched"].nslots
    if C > 1:
        P = dict(P)
        P["stage"] = False
        if not P["arena_smem"] or wsched.LANES * P["es"] * (P["sin"] + na) > wsched.SMEM_BUDGET:
            raise GenerationError(f"{model.name} {alg} {dt}: the cluster arena must fit shared memory")
        P["arena_smem"] = True
    em, sched = P["em"], P["sched"]
    n, nin = P["n"], P["nin"]
    T = "double" if dt == "f64" else "float"
    ar_space = "shared" if P["arena_smem"] else "global"
    out_space = "shared" if P["stage"] else "global"
    AT = "unsigned" if P["arena_smem"] else "unsigned long long"
    OT = "unsigned" if P["stage"] else "unsigned long long"
    ac = '"r"' if P["arena_smem"] else '"l"'
    oc = '"r"' if P["stage"] else '"l"'
    ext = P["ext"]
    src = [
        f"// GENERATED by paper_2109_06976_b200.codegen -- robot {model.name!r}, {alg} {dt}, warp-specialised",
    ] + [f"// variant {v}: {len(p['sched'].task_ops)} tasks in {len(p['sched'].phases)} phases over {sw} warps"
         f"{f' ({C} CTAs)' if C > 1 else ''}; "
         f"critical path {p['sched'].critical_path()} of {p['sched'].total()} ops; {p['sched'].nslots} arena slots"
         for v, p in enumerate(Ps)] + [
        f"// {em.flops} flops per knot (variant 0); arena {ar_space}",
        "#pragma once",
        '#include "rbd_runtime.cuh"',
        f"struct {name or f'Knot_{alg}_{dt}'} {{",
        f"  typedef {T} T;",
        ("  static constexpr int MAP = 1;  // warp-specialised: CTA = 32 knots x W warps" if C == 1 else
         "  static constexpr int MAP = 3;  // warp-specialised over a cluster: C CTAs x W warps on 32 knots"),
        f"  static constexpr int W = {warps}, NDOF = {n}, NIN = {nin}, NSC = {P['nsc']}, NVAR = {len(Ps)}, C = {C};",
        f"  static constexpr int LO = {em.lo}, NP = {em.np};  // input dof window [LO, LO + NP)",
    ] + _input_consts(em.in_layout) + [
        f"  static constexpr int E0 = {ext[0]}, E1 = {ext[1]}, E2 = {ext[2]};",
        f"  static constexpr int SIN = {P['sin']}, NA = {na}, SOUT = {P['sout']};",
        f"  static constexpr bool STAGE = {'true' if P['stage'] else 'false'}, "
        f"ARENA_SMEM = {'true' if P['arena_smem'] else 'false'};",
        f"  static constexpr bool ARENA_GROUP = {'true' if P.get('imports') else 'false'};"
        "  // arena = the group's slice of the split scratch",
        f"  static constexpr int FLOPS = {em.flops};",
        f"  static constexpr int MINB = {int(tuning(model, alg, dt).get('minb', 1))};  // min CTAs per SM (register cap)",
        "  typedef " + AT + " arena_t;",
        "  typedef " + OT + " out_t;",
        "  __device__ __forceinline__ static void prologue(T* s_in, int warp, int lane) {",
    ]
    sc_fn = "rbd_sincos_fast" if tuning(model, alg, dt).get("ws_fast_sincos") else "rbd_sincos"
    k = 0
    for op in em.ops:
        if op[0] == "sincos":
            slot = op[3]
            src.append(f"    if (warp == {k % warps}) {{ T s, c; {sc_fn}(s_in[{slot * 33} + lane], &s, &c); "
                       f"s_in[{(em.in_total + 2 * k) * 33} + lane] = s; s_in[{(em.in_total + 2 * k + 1) * 33} + lane] = c; }}")
            k += 1
    src.append("    (void)s_in; (void)warp; (void)lane;")
    src.append("  }")
    if C == 1:
        src.append("  __device__ __forceinline__ static void run_group(int var, int warp, unsigned a_in, arena_t a_ar, "
                   "out_t a0, out_t a1, out_t a2, unsigned valid) {")
    else:
        src.append("  __device__ __forceinline__ static void run_group(int var, int warp, unsigned a_in, arena_t a_ar, "
                   "const unsigned* a_rem, out_t a0, out_t a1, out_t a2, unsigned valid) {")
    rem_ops = "".join(f', "r"(a_rem[{r}])' for r in range(C)) if C > 1 else ""
    sync = "__syncthreads();" if C == 1 else "rbd_cluster_sync();"
    tn = tuning(model, alg, dt)
    ctab = ConstTable(f"rbd_c_{name or f'Knot_{alg}_{dt}'}", dt)
    multi = len(Ps) > 1
    if multi:
        src.append("    switch (var) {")
    for v, Pv in enumerate(Ps):
        sv, emv = Pv["sched"], Pv["em"]
        if multi:
            src.append(f"    case {v}: {{")
        cta_of = None
        if C > 1:  # value -> CTA rank of the warp producing it
            wof = {t: w for ph in sv.phases for w, ts in enumerate(ph) for t in ts}
            cta_of = {r: wof[t] // warps for r, t in sv.export.items()}
        for p, phase in enumerate(sv.phases):
            src.append(f"    // variant {v} phase {p}")
            src.append("    switch (warp) {")
            for w, tasks in enumerate(phase):
                if not tasks:
                    continue
                body = wsched.ptx_block(sv, tasks, dt, emv.in_total, emv.in_total, ar_space, out_space,
                                        tn["reload_dist"], ctab, cta_of=cta_of, my_cta=w // warps)
                src.append(f"    case {w}:  // {', '.join(tasks)}")
                src.append('      asm volatile("{\\n\\t"')
                for ln in body:
                    src.append(f'        "{ln}\\n\\t"')
                src.append(f'        "}}" :: "r"(a_in), {ac}(a_ar), {oc}(a0), {oc}(a1), {oc}(a2), "r"(valid)'
                           f'{rem_ops} : "memory");')
                src.append("      break;")
            src.append("    default: break;")
            src.append("    }")
            src.append(f"    {sync}")
        if multi:
            src.append("    } break;")
    if multi:
        src.append("    default: break;")
        src.append("    }")
    src.append("    (void)var; (void)a_in; (void)a_ar; (void)a0; (void)a1; (void)a2; (void)valid;")
    src += ["  }", "};", ""]
    decl = ctab.declaration()
    src = src[:5] + decl + src[5:]  # after the #include
    L = dict(nin=nin, ext=ext)
    return "\n".join(src), em.flops, L


def _fs_struct(model, alg, dt, warps, variants, name, fext=False, em=None):
    """Device header of the fine-grained warp-specialised mapping (fsched.py):
    per (column variant, warp) one asm block holding that warp's whole
    program, phases separated by bar.sync; arena in shared memory."""
    from . import fsched
    if em is None:
        em = generate_knot(model, alg, dt, fext=fext)
    n = model.n_dof
    es = 8 if dt == "f64" else 4
    nsc = sum(1 for op in em.ops if op[0] == "sincos")
    sin = em.in_total + 2 * nsc
    ext = [e for _, e in outputs(alg, n)]
    ext += [0] * (3 - len(ext))
    progs = fsched.split_variants(em, variants) if alg in ("gradID", "gradFD") else [em]
    stage = len(progs) == 1 and 33 * es * (sin + sum(ext)) <= 96 * 1024
    budget = (FS_SMEM_BUDGET // (33 * es)) - sin - (sum(ext) if stage else 0)
    scheds = [fsched.FineSchedule(p, warps, max_slots=budget) for p in progs]
    na = max(1, max(S.nslots for S in scheds))
    if na > budget:
        raise GenerationError(f"{model.name} {alg} {dt}: fs arena of {na} slots does not fit shared memory")
    out_space = "shared" if stage else "global"
    T = "double" if dt == "f64" else "float"
    OT = "unsigned" if stage else "unsigned long long"
    oc = '"r"' if stage else '"l"'
    K = name
    ctab = ConstTable(f"rbd_c_{K}", dt)
    src = [
        f"// GENERATED by paper_2109_06976_b200.codegen -- robot {model.name!r}, {alg} {dt}, fine-grained "
        f"warp-specialised ({warps} warps, {len(progs)} column variants)",
    ]
    for v, S in enumerate(scheds):
        src.append(f"// variant {v}: {S.total()} ops in {S.nphases} phases, {S.nslots} arena slots, "
                   f"simulated {S.critical_path()} cycles (delta {S.delta}, window {S.window})")
    src += ["#pragma once", '#include "rbd_runtime.cuh"', "@CTAB@",
            f"struct {K} {{",
            f"  typedef {T} T;",
            "  static constexpr int MAP = 2;  // fine-grained warp-specialised: CTA = 32 knots x W warps",
            f"  static constexpr int W = {warps}, NVAR = {len(progs)}, NDOF = {n}, NIN = {len(em.in_layout)}, "
            f"NSC = {nsc};",
            f"  static constexpr int LO = {em.lo}, NP = {em.np};  // input dof window [LO, LO + NP)",
            ] + _input_consts(em.in_layout) + [
            f"  static constexpr int E0 = {ext[0]}, E1 = {ext[1]}, E2 = {ext[2]};",
            f"  static constexpr int SIN = {sin}, NA = {na}, SOUT = {sum(ext)};",
            f"  static constexpr bool STAGE = {'true' if stage else 'false'};",
            f"  static constexpr int FLOPS = {em.flops};",
            "  static constexpr int MINB = 1;",
            f"  typedef {OT} out_t;",
            "  __device__ __forceinline__ static void prologue(T* s_in, int warp, int lane) {"]
    sc_fn = "rbd_sincos_fast" if tuning(model, alg, dt).get("ws_fast_sincos") else "rbd_sincos"
    k = 0
    for op in em.ops:
        if op[0] == "sincos":
            slot = op[3]
            src.append(f"    if (warp == {k % warps}) {{ T s, c; {sc_fn}(s_in[{slot * 33} + lane], &s, &c); "
                       f"s_in[{(em.in_total + 2 * k) * 33} + lane] = s; s_in[{(em.in_total + 2 * k + 1) * 33} + lane] = c; }}")
            k += 1
    src += ["    (void)s_in; (void)warp; (void)lane;", "  }",
            "  __device__ __forceinline__ static void run(int var, int warp, unsigned a_in, unsigned a_ar, "
            "out_t a0, out_t a1, out_t a2, unsigned valid) {",
            f"    switch (var * {warps} + warp) {{"]
    for v, S in enumerate(scheds):
        for w in range(warps):
            body = fsched.ptx_warp(S, w, dt, em.in_total, out_space, ctab,
                                   sincos_slots=[op[3] for op in em.ops if op[0] == "sincos"])
            src.append(f"    case {v * warps + w}:  // variant {v}, warp {w}")
            src.append('      asm volatile("{\\n\\t"')
            for ln in body:
                src.append(f'        "{ln}\\n\\t"')
            src.append(f'        "}}" :: "r"(a_in), "r"(a_ar), {oc}(a0), {oc}(a1), {oc}(a2), "r"(valid) : "memory");')
            src.append("      break;")
    src += ["    default: break;", "    }", "  }", "};", ""]
    text = "\n".join(src).replace("@CTAB@", "\n".join(ctab.declaration()))
    return text, em.flops, dict(nin=len(em.in_layout), ext=ext)


FS_SMEM_BUDGET = 200 * 1024  # dynamic shared memory per CTA the fs mapping may use


def mapping(model, alg, dt):
    """'thread' (one knot per thread) or 'ws' (warp-specialised), from tuning."""
    return tuning(model, alg, dt).get("map", "thread")


def host_sources(model, algorithms=ALGORITHMS, dtypes=DTYPES):
    """TEST-ONLY: plain C++ one-knot programs for the host harness
    (Knot_<alg>_<dt>, and Knot_<alg>_<dt>_X with the f_ext input)."""
    files = {}
    for alg in algorithms:
        for dt in dtypes:
            for fx in ((False, True) if alg in FEXT_ALGORITHMS else (False,)):
                em = generate_knot(model, alg, dt, fext=fx)
                L = _layout(model, alg, dt, em, device=False)
                name = f"Knot_{alg}_{dt}" + ("_X" if fx else "")
                src = ["#pragma once", '#include "rbd_runtime.cuh"'] + _struct_head(model, alg, dt, L, em.flops, name) + [
                    "  static inline void run(const T* __restrict__ iq, const T* __restrict__ iqd,",
                    "                         const T* __restrict__ iu, const T* __restrict__ ifx,",
                    "                         T* __restrict__ o0, T* __restrict__ o1, T* __restrict__ o2) {",
                    "    (void)iqd; (void)iu; (void)ifx; (void)o1; (void)o2;",
                ] + ["    " + ln for ln in cpp_body(em, L["n"])] + ["  }", "};", ""]
                files[f"host_{alg}_{dt}{'_X' if fx else ''}.h"] = "\n".join(src)
    files["host_all.h"] = "\n".join(["#pragma once"] + [f'#include "{f}"' for f in sorted(files)]) + "\n"
    return files


def _launch_unit(alg, dt, tag, K, text, rollout=False):
    """Translation unit of one kernel: its struct + the internal launcher
    (+ the fused-rollout launcher of a whole-robot warp-specialised FD /
    gradFD program)."""
    extra = []
    if rollout:
        extra = [
            f'extern "C" int rbd__rollout_{alg}_{dt}(void* q, void* qd, const void* tau, void* o0, void* o1, void* o2,',
            "                                int64_t B, int32_t H, double dt, void* stream) {",
            f"  return rbd_launch_rollout<{K}>(q, qd, tau, o0, o1, o2, B, H, dt, stream);",
            "}",
        ]
    return "\n".join([
        text.replace("#pragma once\n", ""),
        f'extern "C" int rbd__launch_{alg}_{dt}_{tag}(const void* q, const void* qd, const void* u, const void* fx,',
        "                                void* o0, void* o1, void* o2, int64_t N, void* stream) {",
        f"  return rbd_launch_kernel<{K}>(q, qd, u, fx, o0, o1, o2, N, stream);",
        "}",
    ] + extra + [""])


def _ws_split_unit(model, alg, dt, tag, K, tn):
    """Small-batch split (wsched.split_programs) as two warp-specialised
    kernels launched back to back: KA = the big tree's prefix (exports to a
    per-device [N][nx] scratch, qdd), KB = CTA-row variants of its gradient
    columns (the scratch as 4th input) and of the other root trees."""
    from . import wsched
    n = model.n_dof
    pre, progs, nx = wsched.split_programs(model, alg, dt, int(tn["wsplit_groups"]))
    ta, _, _ = _ws_struct(model, alg, dt, int(tn["wsplit_warps"]), K + "A", em=pre,
                          ext=[nx, n if alg == "gradFD" else 0, 0])
    tb, fl, L = _ws_struct(model, alg, dt, int(tn["wc_warps"]), K + "B", progs=progs)
    maxn = int(tn["wsplit_max_n"])
    unit = "\n".join([
        ta.replace("#pragma once\n", ""), tb.replace("#pragma once\n", ""),
        f'extern "C" int rbd__launch_{alg}_{dt}_{tag}(const void* q, const void* qd, const void* u, const void* fx,',
        "                                void* o0, void* o1, void* o2, int64_t N, void* stream) {",
        f"  (void)fx;",
        f"  return rbd_launch_ws_split<{K}A, {K}B, {maxn}>(q, qd, u, o0, o1, o2, N, stream);",
        "}",
        "",
    ])
    return unit, fl, L


def _big_part_unit(model, alg, dt, tag, K, tn, trees, zero_fill, fx):
    """A part whose one-knot program does not fit a thread.  Gradient
    programs are split (`split_columns`): a thread-per-knot prefix kernel
    exporting to an L2-resident scratch + a thread-per-knot column kernel
    whose register plan reloads the imports from that scratch; other
    algorithms run warp-specialised as a whole."""
    if alg in ("gradID", "gradFD") and tn.get("split", True):
        em = generate_knot(model, alg, dt, trees, zero_fill, fext=fx, lowmem=True)
        by_task = tn.get("split_by_task") or False
        pre, progs, nx = split_columns(em, by_task=by_task)
        pf = {"park": False, "prefetch_dist": int(tn.get("split_pf_dist", 96)),
              "prefetch_slack": int(tn.get("split_pf_slack", 12)), "ra_budget": int(tn.get("split_budget", 0))}
        tmem = int(tn.get("split_tmem", 0))  # imports homed in tensor memory (column kernel, 128-knot CTAs)
        if tmem:
            pf["bk"] = int(tn.get("split_bk", 128))  # 4k warps per CTA over the TMEM lane quadrants
        try:
            ta, _, _ = _knot_struct(model, alg, dt, K + "A", em=pre, nx=nx)
            # knots per launch pair: large enough that the prefix kernel fills
            # the GPU, small enough that the scratch mostly stays in L2
            chunk = int(tn.get("split_chunk") or 32768)
            ta = ta.replace(f"  static constexpr int NX = {nx};",
                            f"  static constexpr int NX = {nx};\n  static constexpr int CHUNK = {chunk};"
                            "  // knots per split launch pair")
            if by_task:
                # one program per gradient column (short code, every warp of a
                # CTA on the same column); a column whose outputs are all
                # structural zeros (memset) has no work
                progs = [p for p in progs if any(op[0] != "st" or not isinstance(op[3], float)
                                                 for op, t in zip(p.ops, p.tasks) if t.startswith("grad."))]
                tb = _multi_knot_struct(model, alg, dt, K + "B", progs, nx, pf, tmem=tmem)
            else:
                # all columns in one program; outputs stored as they are produced
                tb, _, _ = _knot_struct(model, alg, dt, K + "B", em=progs, nx=nx, over=pf, tmem=tmem)
            return "\n".join([
                ta.replace("#pragma once\n", ""), tb.replace("#pragma once\n", ""),
                f'extern "C" int rbd__launch_{alg}_{dt}_{tag}(const void* q, const void* qd, const void* u, '
                "const void* fx,",
                "                                void* o0, void* o1, void* o2, int64_t N, void* stream) {",
                f"  return rbd_launch_split<{K}A, {K}B>(q, qd, u, fx, o0, o1, o2, N, stream);",
                "}",
                f'extern "C" int rbd__fork_{alg}_{dt}_{tag}(const void* q, const void* qd, const void* u, '
                "const void* fx,",
                "                                void* o0, void* o1, void* o2, int64_t N, void* stream) {",
                f"  return rbd_launch_split<{K}A, {K}B>(q, qd, u, fx, o0, o1, o2, N, stream, false);",
                "}",
                f'extern "C" int rbd__join_{alg}_{dt}_{tag}(void* stream) {{',
                f"  return rbd_split_join<{K}A, {K}B>(stream);",
                "}",
                "",
            ])
        except GenerationError:
            pass
    text, _, _ = _ws_struct(model, alg, dt, int(tn["warps"]), K, trees=trees, zero_fill=zero_fill, fext=fx)
    return _launch_unit(alg, dt, tag, K, text)


def generate_sources(model, algorithms=ALGORITHMS, dtypes=DTYPES):
    """{file name: text} of the per-robot library plus {(alg, dtype): flops}.

    k_<alg>_<dt>_<tag>.cu  one kernel (struct with the one-knot program + its
                           launcher); tag T = thread per knot, W = warp-
                           specialised, P<k> = part k (root-tree subset), with
                           an X suffix for the f_ext variant
    main.cu                dispatch (batch size -> mapping), typed C-ABI
                           entries rbd_<alg>_<dt>[_fext], rbd_get_info,
                           rbd_launch[_fext], host sessions
    Separate translation units let nvcc/ptxas run in parallel.
    """
    n = model.n_dof
    fp = model_hash(model)
    files, flops, table = {}, {}, {}
    dispatch = []
    rollouts = set()
    zc_direct = {}  # (alg, dt, fext) -> the host path's small-batch launcher stages its outputs
    sig = "(const void*, const void*, const void*, const void*, void*, void*, void*, int64_t, void*);"
    args = "(q, qd, u, fx, o0, o1, o2, N, stream)"
    for alg in algorithms:
        for dt in dtypes:
            T = "double" if dt == "f64" else "float"
            tn = tuning(model, alg, dt)
            maps = list(tn["maps"])
            for fx in ((False, True) if alg in FEXT_ALGORITHMS else (False,)):
                X = "X" if fx else ""
                tags = []
                for mp in maps:
                    if mp == "wsplit" and (fx or alg not in ("gradID", "gradFD")):
                        continue
                    tag = {"ws": "W", "fs": "F", "wc": "C", "wsplit": "S"}.get(mp, "T") + X
                    K = f"Knot_{alg}_{dt}_{tag}"
                    if mp == "wsplit":
                        unit, fl, L = _ws_split_unit(model, alg, dt, tag, K, tn)
                        files[f"k_{alg}_{dt}_{tag}.cu"] = unit
                        tags.append(tag)
                        continue
                    if mp == "wc":
                        text, fl, L = _ws_struct(model, alg, dt, int(tn["wc_warps"]), K, fext=fx,
                                                 variants=int(tn["wc_variants"]), cluster=int(tn["wc_cluster"]))
                    elif mp == "fs":
                        text, fl, L = _fs_struct(model, alg, dt, int(tn["fs_warps"]), int(tn["fs_variants"]), K,
                                                 fext=fx)
                    elif mp == "ws":
                        text, fl, L = _ws_struct(model, alg, dt, int(tn["warps"]), K, fext=fx,
                                                 variants=int(tn.get("ws_variants", 0)))
                    else:
                        text, fl, L = _knot_struct(model, alg, dt, K, fext=fx)
                    if not fx:
                        flops[(alg, dt)] = fl
                    table[(alg, dt, fx)] = (L["nin"], L["ext"], 8 if dt == "f64" else 4)
                    ro = (mp == "ws" and not fx and alg in ("FD", "gradFD") and int(tn.get("ws_variants", 0)) <= 1)
                    files[f"k_{alg}_{dt}_{tag}.cu"] = _launch_unit(alg, dt, tag, K, text, rollout=ro)
                    if ro:
                        rollouts.add((alg, dt))
                    tags.append(tag)
                # large batches of a robot with several root trees: one kernel per
                # part (a group of trees), each mapped on its own (thread per knot
                # when its register plan fits, else warp-specialised); cross-part
                # structural zeros by a coalesced memset ("zero_memset") or by part 0
                parts = tn.get("parts") or []
                zf = not tn.get("zero_memset")
                ptags, split_tags = [], []
                for pi, trees in enumerate(parts):
                    tag = f"P{pi}{X}"
                    K = f"Knot_{alg}_{dt}_{tag}"
                    try:
                        po = tn.get("part_over") or {}
                        text, fl, L = _knot_struct(model, alg, dt, K, trees=tuple(trees), zero_fill=zf and pi == 0,
                                                   fext=fx, over=po.get(pi, po.get(str(pi))))
                        if (L["minb"] * L["bk"] < 32 * int(tn.get("min_warps", 4)) and alg in ("gradID", "gradFD")
                                and tn.get("split")):
                            raise GenerationError("thread-per-knot occupancy too low; split the program")
                        files[f"k_{alg}_{dt}_{tag}.cu"] = _launch_unit(alg, dt, tag, K, text)
                    except GenerationError:
                        files[f"k_{alg}_{dt}_{tag}.cu"] = _big_part_unit(model, alg, dt, tag, K, tn, tuple(trees),
                                                                         zf and pi == 0, fx)
                        if "rbd__fork_" in files[f"k_{alg}_{dt}_{tag}.cu"]:
                            split_tags.append(tag)
                    ptags.append(tag)
                for tag in tags + ptags:
                    dispatch.append(f'extern "C" int rbd__launch_{alg}_{dt}_{tag}{sig}')
                for tag in split_tags:
                    dispatch.append(f'extern "C" int rbd__fork_{alg}_{dt}_{tag}{sig}')
                    dispatch.append(f'extern "C" int rbd__join_{alg}_{dt}_{tag}(void*);')
                if ptags:
                    # split parts run their pipeline on side streams while the
                    # other parts (independent root trees) run on the caller's
                    seq = " ".join([f"if ((rc = rbd__fork_{alg}_{dt}_{t}{args}) != 0) return rc;" for t in split_tags]
                                   + [f"if ((rc = rbd__launch_{alg}_{dt}_{t}{args}) != 0) return rc;"
                                      for t in ptags if t not in split_tags]
                                   + [f"if ((rc = rbd__join_{alg}_{dt}_{t}(stream)) != 0) return rc;"
                                      for t in split_tags])
                    zs = ""
                    if not zf and alg in ("Minv", "gradID", "gradFD"):
                        es = 8 if dt == "f64" else 4
                        zs = (f"if ((rc = (int)cudaMemsetAsync(o0, 0, (size_t)N * {n * n * es}, "
                              f"(cudaStream_t)stream)) != 0) return rc; ")
                        if alg != "Minv":
                            zs += (f"if ((rc = (int)cudaMemsetAsync(o1, 0, (size_t)N * {n * n * es}, "
                                   f"(cudaStream_t)stream)) != 0) return rc; ")
                    big = f"[&]() {{ int rc; {zs}{seq} return 0; }}()"
                else:
                    big = f"rbd__launch_{alg}_{dt}_{'T' if 'thread' in maps else 'W'}{X}{args}"
                if "ws" in maps and (ptags or "thread" in maps):
                    pick = f"N <= {int(tn['ws_max_n'])} ? rbd__launch_{alg}_{dt}_W{X}{args} : {big}"
                elif ptags:
                    pick = big
                else:
                    pick = f"rbd__launch_{alg}_{dt}_{'W' if maps[0] == 'ws' else 'T'}{X}{args}"
                if "fs" in maps:
                    # small batches: the fine-grained schedule (lowest latency)
                    pick = f"N <= {int(tn['fs_max_n'])} ? rbd__launch_{alg}_{dt}_F{X}{args} : ({pick})"
                # the small-batch host path (zero-copy outputs into pinned host
                # memory) prefers kernels that stage their outputs (coalesced
                # PCIe writes) when the robot's tuning says so ("zc_variants")
                host_pick = pick
                if "wsplit" in maps and not fx and alg in ("gradID", "gradFD"):
                    # mid-size batches of a big tree: prefix once, then the column variants
                    pick = f"N <= {int(tn['wsplit_max_n'])} ? rbd__launch_{alg}_{dt}_S{args} : ({pick})"
                if not tn.get("zc_variants", True):
                    host_pick = pick
                if "wc" in maps:
                    # small batches: one knot group's tasks over a cluster / several CTA rows
                    pick = f"N <= {int(tn['wc_max_n'])} ? rbd__launch_{alg}_{dt}_C{X}{args} : ({pick})"
                if tn.get("zc_variants", True):
                    host_pick = pick
                dispatch += [
                    f'extern "C" int rbd__launch_{alg}_{dt}{"_fext" if fx else ""}(const void* q, const void* qd, '
                    "const void* u, const void* fx,",
                    "                                void* o0, void* o1, void* o2, int64_t N, void* stream) {",
                    f"  return {pick};",
                    "}",
                    f'extern "C" int rbd__launch_{alg}_{dt}{"_fext" if fx else ""}_host(const void* q, const void* qd, '
                    "const void* u, const void* fx,",
                    "                                void* o0, void* o1, void* o2, int64_t N, void* stream) {",
                    f"  return {host_pick};",
                    "}",
                ]
                zc_direct[(alg, dt, fx)] = host_pick != pick
            dispatch += [
                f'extern "C" int rbd_{alg}_{dt}(const {T}* q, const {T}* qd, const {T}* u, {T}* o0,',
                f"                         {T}* o1, {T}* o2, int64_t N, void* stream) {{",
                f"  return rbd__launch_{alg}_{dt}(q, qd, u, nullptr, o0, o1, o2, N, stream);",
                "}",
            ]
            if alg in FEXT_ALGORITHMS:
                dispatch += [
                    f'extern "C" int rbd_{alg}_{dt}_fext(const {T}* q, const {T}* qd, const {T}* u, '
                    f"const {T}* f_ext, {T}* o0,",
                    f"                         {T}* o1, {T}* o2, int64_t N, void* stream) {{",
                    f"  return rbd__launch_{alg}_{dt}_fext(q, qd, u, f_ext, o0, o1, o2, N, stream);",
                    "}",
                ]
    main = [
        f"// GENERATED by paper_2109_06976_b200.codegen -- robot {model.name!r}, n_dof={n}",
        f"// model fingerprint sha256 {fp}",
        "#define RBD_MAIN_TU 1",
        '#include "rbd_runtime.cuh"',
        "",
    ]
    main += dispatch
    # fused rollouts (rbd_rollout): FD / gradFD over a horizon in one launch
    for (alg, dt) in sorted(rollouts):
        main.append(f'extern "C" int rbd__rollout_{alg}_{dt}(void*, void*, const void*, void*, void*, void*, int64_t, '
                    "int32_t, double, void*);")
    main += [
        'extern "C" int rbd_rollout(int alg, int dtype, void* q, void* qd, const void* tau, void* qdd, void* dq,',
        "                           void* dqd, int64_t B, int32_t H, double dt, void* stream) {",
    ]
    for (alg, dt) in sorted(rollouts):
        a, d = _ALG_ENUM[alg], (1 if dt == "f64" else 0)
        call = (f"rbd__rollout_FD_{dt}(q, qd, tau, qdd, nullptr, nullptr, B, H, dt, stream)" if alg == "FD" else
                f"rbd__rollout_gradFD_{dt}(q, qd, tau, dq, dqd, qdd, B, H, dt, stream)")
        main.append(f"  if (alg == {a} && dtype == {d}) return {call};")
    main += ["  (void)q; (void)qd; (void)tau; (void)qdd; (void)dq; (void)dqd; (void)B; (void)H; (void)dt; (void)stream;",
             "  return RBD_EINVAL;", "}"]
    main += [
        "",
        "static int rbd_ndof() { return %d; }" % n,
        "static const rbd_entry* rbd_entry_for(int alg, int dtype, int fext) {",
        "  static const rbd_entry table[5][2][2] = {",
    ]
    for alg in ALGORITHMS:
        row = []
        for dt in DTYPES:
            pair = []
            for fx in (False, True):
                if (alg, dt, fx) in table:
                    nin, ext, es = table[(alg, dt, fx)]
                    fn = f"rbd__launch_{alg}_{dt}{'_fext' if fx else ''}"
                    tn = tuning(model, alg, dt)
                    cmax = max(int(tn["wc_max_n"]) if "wc" in tn["maps"] else 0,
                               int(tn["wsplit_max_n"]) if "wsplit" in tn["maps"] and not fx else 0)
                    if zc_direct.get((alg, dt, fx)):
                        cmax = 0  # the host launcher runs output-staging kernels: zero-copy outputs
                    pair.append(f"{{&{fn}, {nin}, {ext[0]}, {ext[1]}, {ext[2]}, {es}, {cmax}, &{fn}_host}}")
                else:
                    pair.append("{nullptr, 0, 0, 0, 0, 0, 0, nullptr}")
            row.append("{" + ", ".join(pair) + "}")
        main.append("    {" + ", ".join(row) + "},")
    main += [
        "  };",
        "  if (alg < 0 || alg > 4 || dtype < 0 || dtype > 1 || fext < 0 || fext > 1) return nullptr;",
        "  return table[alg][dtype][fext].fn ? &table[alg][dtype][fext] : nullptr;",
        "}",
        "",
        'extern "C" int rbd_get_info(rbd_info* out) {',
        "  if (!out) return RBD_EINVAL;",
        "  out->abi_version = RBD_ABI_VERSION;",
        f"  out->n_dof = {n};",
        f"  out->n_frames = {model.n_frames};",
        f"  out->n_trees = {len(model.roots())};",
        f"  out->knots_per_block = {knots_per_block(model, 'gradFD', 'f64')};",
        "  out->reserved = 0;",
        f'  out->robot = "{model.name}";',
        f'  out->fingerprint = "{fp}";',
        "  return 0;",
        "}",
        "",
    ]
    files["main.cu"] = "\n".join(main)
    return files, flops
