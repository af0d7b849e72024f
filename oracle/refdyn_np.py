"""CPU oracle: numpy restatement of the reference dynamics (TEST INFRASTRUCTURE).

This module is the checker, never the product.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may import it.
The product path (`paper_2109_06976_b200`) never imports anything under
`oracle/` and has no CPU fallback.

Each function restates one function of the reference `rbdgen/refdyn.py`
(cited per function) in per-knot numpy, with the same operation structure
(dense 6x6 transforms per frame, per-column gradient loops), so that timing
it on the host cores measures the reference's own CPU path.

Pinning: the reference ships no golden vectors.  `tests/golden/make_golden.py`
imports the reference (`/root/reference/pkg/src/rbdgen`) in the build
container and records its outputs for every bundled robot and algorithm on
seeded inputs; `tests/test_oracle.py` checks this module against those
fixtures (fp64, 1e-12 relative) and against the SPEC known-answer tests.

Conventions (reference `refdyn.py:1-13`): spatial vectors [angular; linear],
gravity enters as base acceleration a0 = [0, 0, 0, -g], f_ext per frame in
link coordinates, subtracted from the body force.
"""

import numpy as np


# -- spatial pieces (reference spatial.py) ------------------------------------

def _skew(w):
    return np.array([[0.0, -w[2], w[1]], [w[2], 0.0, -w[0]], [-w[1], w[0], 0.0]])


def motion_cross(v):
    """v x (reference `spatial.py:45-65`): [[w x, 0], [l x, w x]]."""
    out = np.zeros((6, 6))
    W, L = _skew(v[:3]), _skew(v[3:])
    out[:3, :3] = W
    out[3:, 3:] = W
    out[3:, :3] = L
    return out


def force_cross(v):
    """v x* = -(v x)^T (reference `spatial.py:68-70`)."""
    return -motion_cross(v).T


def _rodrigues(u, ang):
    K = _skew(u)
    return np.eye(3) + np.sin(ang) * K + (1.0 - np.cos(ang)) * (K @ K)


def joint_xform(joint, qi):
    """Dense parent->child motion transform (reference `spatial.py:96-102`,
    `:180-196`): [[E, 0], [-E skew(r), E]]."""
    R0 = np.asarray(joint.origin_rotation, dtype=float)
    r = np.asarray(joint.origin_translation, dtype=float)
    if joint.kind == "revolute":
        E = _rodrigues(np.asarray(joint.axis, dtype=float), qi).T @ R0.T
    elif joint.kind == "prismatic":
        E = R0.T.copy()
        r = r + R0 @ (qi * np.asarray(joint.axis, dtype=float))
    else:
        E = R0.T.copy()
    X = np.zeros((6, 6))
    X[:3, :3] = E
    X[3:, 3:] = E
    X[3:, :3] = -E @ _skew(r)
    return X


def joint_subspace(joint):
    """S (reference `spatial.py:199-206`)."""
    u = np.asarray(joint.axis, dtype=float)
    z = np.zeros(3)
    return np.concatenate([u, z]) if joint.kind == "revolute" else np.concatenate([z, u])


def body_inertia(ine):
    """6x6 spatial inertia (reference `spatial.py:158-166`)."""
    C = _skew(ine.com)
    m = float(ine.mass)
    I = np.zeros((6, 6))
    I[:3, :3] = np.asarray(ine.inertia_about_com) + m * (C @ C.T)
    I[:3, 3:] = m * C
    I[3:, :3] = m * C.T
    I[3:, 3:] = m * np.eye(3)
    return I


def _frames(model, q):
    """reference `refdyn.py:41-47`."""
    n = len(model.parent)
    X = [joint_xform(model.joints[i], q[i]) for i in range(n)]
    S = [joint_subspace(model.joints[i]) for i in range(n)]
    I = [body_inertia(model.inertias[i]) for i in range(n)]
    return X, S, I


def _a0(model):
    """reference `refdyn.py:50-52`."""
    g = np.asarray(model.gravity, dtype=float)
    return np.concatenate([np.zeros(3), -g])


def check_state(model, *vecs):
    """reference `refdyn.py:31-38`."""
    n = model.n_dof
    for v in vecs:
        v = np.asarray(v)
        if v.shape != (n,):
            raise ValueError(f"state vector has shape {v.shape}, expected ({n},)")
        if not np.all(np.isfinite(v)):
            raise ValueError("state vector contains non-finite entries")


# -- algorithms (reference refdyn.py) -------------------------------------------

def newton_euler(model, q, qd, qdd, f_ext=None):
    """Both RNEA sweeps (reference `refdyn.py:55-88`): returns v, a, f
    (f accumulated by the backward sweep) and tau."""
    n = len(model.parent)
    X, S, I = _frames(model, q)
    a0 = _a0(model)
    v = np.zeros((n, 6))
    a = np.zeros((n, 6))
    f = np.zeros((n, 6))
    for i in range(n):
        p = model.parent[i]
        vj = S[i] * qd[i]
        if p < 0:
            v[i] = vj
            a[i] = X[i] @ a0
        else:
            v[i] = X[i] @ v[p] + vj
            a[i] = X[i] @ a[p]
        a[i] = a[i] + S[i] * qdd[i] + motion_cross(v[i]) @ vj
        f[i] = I[i] @ a[i] + force_cross(v[i]) @ (I[i] @ v[i])
        if f_ext is not None:
            f[i] = f[i] - np.asarray(f_ext[i])
    tau = np.zeros(n)
    for i in range(n - 1, -1, -1):
        tau[i] = S[i] @ f[i]
        p = model.parent[i]
        if p >= 0:
            f[p] = f[p] + X[i].T @ f[i]
    return v, a, f, tau


def rnea(model, q, qd, qdd, f_ext=None):
    """Inverse dynamics (reference `refdyn.py:91-94`)."""
    check_state(model, q, qd, qdd)
    return newton_euler(model, q, qd, qdd, f_ext)[3]


def bias_force(model, q, qd, f_ext=None):
    """rnea at qdd = 0 (reference `refdyn.py:97-100`)."""
    check_state(model, q, qd)
    return rnea(model, q, qd, np.zeros(model.n_dof), f_ext)


def crba_mass_matrix(model, q):
    """Composite-rigid-body mass matrix (reference `refdyn.py:103-125`), an
    independent check of minv_direct."""
    check_state(model, q)
    n = len(model.parent)
    X, S, I = _frames(model, q)
    Ic = [M.copy() for M in I]
    H = np.zeros((n, n))
    for i in range(n - 1, -1, -1):
        p = model.parent[i]
        if p >= 0:
            Ic[p] = Ic[p] + X[i].T @ Ic[i] @ X[i]
        fh = Ic[i] @ S[i]
        H[i, i] = S[i] @ fh
        j = i
        while model.parent[j] >= 0:
            fh = X[j].T @ fh
            j = model.parent[j]
            H[i, j] = H[j, i] = S[j] @ fh
    return H


def _subtree(model, i):
    out, member = [i], {i}
    for c in range(i + 1, len(model.parent)):
        if model.parent[c] in member:
            out.append(c)
            member.add(c)
    return out


def minv_direct(model, q):
    """Direct inverse mass matrix by the articulated-body recursion
    (reference `refdyn.py:128-169`)."""
    check_state(model, q)
    n = len(model.parent)
    X, S, I = _frames(model, q)
    IA = [M.copy() for M in I]
    F = np.zeros((n, 6, n))
    U = np.zeros((n, 6))
    Dinv = np.zeros(n)
    Mi = np.zeros((n, n))
    for i in range(n - 1, -1, -1):
        p = model.parent[i]
        U[i] = IA[i] @ S[i]
        Dinv[i] = 1.0 / (S[i] @ U[i])
        sub = _subtree(model, i)
        Mi[i, i] = Dinv[i]
        Mi[i, sub] = Mi[i, sub] - Dinv[i] * (S[i] @ F[i][:, sub])
        if p >= 0:
            F[p][:, sub] = F[p][:, sub] + X[i].T @ (F[i][:, sub] + np.outer(U[i], Mi[i, sub]))
            IA[p] = IA[p] + X[i].T @ ((IA[i] - np.outer(U[i], Dinv[i] * U[i])) @ X[i])
    for i in range(n):
        p = model.parent[i]
        if p >= 0:
            t = X[i] @ F[p][:, i:]
            Mi[i, i:] = Mi[i, i:] - Dinv[i] * (U[i] @ t)
            F[i][:, i:] = np.outer(S[i], Mi[i, i:]) + t
        else:
            F[i][:, i:] = np.outer(S[i], Mi[i, i:])
    for i in range(n):
        Mi[i + 1:, i] = Mi[i, i + 1:]
    return Mi


def forward_dynamics(model, q, qd, tau, f_ext=None):
    """qdd = Minv (tau - c) (reference `refdyn.py:172-175`)."""
    check_state(model, q, qd, tau)
    return minv_direct(model, q) @ (np.asarray(tau, dtype=float) - bias_force(model, q, qd, f_ext))


def rnea_grad(model, q, qd, qdd, f_ext=None):
    """(dtau/dq, dtau/dqd) by differentiating both sweeps
    (reference `refdyn.py:178-239`)."""
    check_state(model, q, qd, qdd)
    n = len(model.parent)
    X, S, I = _frames(model, q)
    a0 = _a0(model)
    v, a, f, _ = newton_euler(model, q, qd, qdd, f_ext)
    # [kind][frame] -> (6, n) column blocks; kind 0 = q, 1 = qd
    dv = np.zeros((2, n, 6, n))
    da = np.zeros((2, n, 6, n))
    df = np.zeros((2, n, 6, n))
    for i in range(n):
        p = model.parent[i]
        vj = S[i] * qd[i]
        if p < 0:
            xv = np.zeros(6)
            xa = X[i] @ a0
        else:
            xv = X[i] @ v[p]
            xa = X[i] @ a[p]
            for k in range(2):
                dv[k, i] = X[i] @ dv[k, p]
                da[k, i] = X[i] @ da[k, p]
        dv[0, i][:, i] += motion_cross(xv) @ S[i]
        dv[1, i][:, i] += S[i]
        for k in range(2):
            for c in range(n):
                da[k, i][:, c] += motion_cross(dv[k, i][:, c]) @ vj
        da[0, i][:, i] += motion_cross(xa) @ S[i]
        da[1, i][:, i] += motion_cross(v[i]) @ S[i]
        Iv = I[i] @ v[i]
        vxI = force_cross(v[i]) @ I[i]
        for k in range(2):
            df[k, i] = I[i] @ da[k, i] + vxI @ dv[k, i]
            for c in range(n):
                df[k, i][:, c] += force_cross(dv[k, i][:, c]) @ Iv
    out = np.zeros((2, n, n))
    for i in range(n - 1, -1, -1):
        for k in range(2):
            out[k, i] = S[i] @ df[k, i]
        p = model.parent[i]
        if p >= 0:
            for k in range(2):
                df[k, p] = df[k, p] + X[i].T @ df[k, i]
            df[0, p][:, i] += X[i].T @ (force_cross(S[i]) @ f[i])
    return out[0], out[1]


def fd_grad(model, q, qd, tau, f_ext=None):
    """(dqdd/dq, dqdd/dqd) = -Minv dID at qdd = FD(q, qd, tau)
    (reference `refdyn.py:242-249`)."""
    check_state(model, q, qd, tau)
    Mi = minv_direct(model, q)
    qdd = Mi @ (np.asarray(tau, dtype=float) - bias_force(model, q, qd, f_ext))
    dq, dqd = rnea_grad(model, q, qd, qdd, f_ext)
    return -Mi @ dq, -Mi @ dqd


def finite_diff(fn, x, h):
    """Central-difference Jacobian (reference `refdyn.py:252-262`)."""
    x = np.asarray(x, dtype=float)
    cols = []
    for j in range(x.size):
        e = np.zeros_like(x)
        e[j] = h
        cols.append((np.asarray(fn(x + e)) - np.asarray(fn(x - e))) / (2.0 * h))
    return np.stack(cols, axis=1)


# -- per-algorithm knot evaluation in the operator's I/O naming -----------------
# (reference schedule.py:208-226 input/output segment names)

ALGORITHMS = ("ID", "Minv", "FD", "gradID", "gradFD")


def evaluate(model, alg, q, qd=None, u=None, f_ext=None):
    """One knot of `alg`; returns {output name: flat array} like
    `interp.interpret` (reference `interp.py:83-86`).  f_ext: (n, 6) per-link
    external forces as refdyn takes them (refdyn.py:79-80)."""
    if alg == "ID":
        return {"tau_out": rnea(model, q, qd, u, f_ext)}
    if alg == "Minv":
        return {"minv_out": minv_direct(model, q).ravel()}
    if alg == "FD":
        return {"qdd_out": forward_dynamics(model, q, qd, u, f_ext)}
    if alg == "gradID":
        dq, dqd = rnea_grad(model, q, qd, u, f_ext)
        return {"dq_out": dq.ravel(), "dqd_out": dqd.ravel()}
    if alg == "gradFD":
        Mi = minv_direct(model, q)
        qdd = Mi @ (np.asarray(u, dtype=float) - bias_force(model, q, qd, f_ext))
        dq, dqd = rnea_grad(model, q, qd, qdd, f_ext)
        return {"dq_out": (-Mi @ dq).ravel(), "dqd_out": (-Mi @ dqd).ravel(), "qdd_out": qdd}
    raise ValueError(f"unknown algorithm {alg!r}")


def evaluate_batch(model, alg, q, qd=None, u=None, f_ext=None):
    """Loop `evaluate` over the leading knot axis; returns {name: (N, extent)}.
    f_ext: (N, n, 6) or None."""
    N = q.shape[0]
    outs = None
    for k in range(N):
        r = evaluate(model, alg, q[k], None if qd is None else qd[k], None if u is None else u[k],
                     None if f_ext is None else np.asarray(f_ext[k]).reshape(-1, 6))
        if outs is None:
            outs = {nm: np.zeros((N,) + np.shape(v)) for nm, v in r.items()}
        for nm, v in r.items():
            outs[nm][k] = v
    return outs
