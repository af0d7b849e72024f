"""Golden vectors from the reference implementation itself.

Imports the reference package (`/root/reference/pkg/src/rbdgen`, pure Python,
numpy only) in the build container and records, for every bundled robot:

* the parsed model (parent indices, joint kinds/axes/origins, inertias) as the
  reference's parser produces it (`urdf.py:180`), to pin our own parser;
* seeded inputs (q ~ U(-pi, pi), qd ~ U(-1, 1), u ~ U(-1, 1),
  seed 0) and the reference outputs of rnea / minv_direct /
  forward_dynamics / rnea_grad / fd_grad (`refdyn.py:91-249`), in the
  operator's I/O naming (`schedule.py:208-226`);
* for gradFD also qdd (the kernel's extra output);
* the same four f_ext-taking entries with seeded per-link external forces
  f_ext ~ U(-1, 1), shape (N, n, 6), seed 2 (refdyn.py:79-80), keys "fext.*".

The reference cannot travel to the GPU box, so the fixtures are committed:

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from rbdgen import models, refdyn  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
N_KNOTS = 16


def inputs(n, N, seed=0):
    rng = np.random.default_rng(seed)
    q = rng.uniform(-np.pi, np.pi, size=(N, n))
    qd = rng.uniform(-1.0, 1.0, size=(N, n))
    u = rng.uniform(-1.0, 1.0, size=(N, n))
    return q, qd, u


def main():
    for name in models.names():
        m = models.load(name)
        n = m.n_dof
        q, qd, u = inputs(n, N_KNOTS)
        rec = {
            "parent": np.array(m.parent),
            "kind": np.array([j.kind for j in m.joints]),
            "axis": np.array([j.axis for j in m.joints]),
            "origin_rotation": np.array([j.origin_rotation for j in m.joints]),
            "origin_translation": np.array([j.origin_translation for j in m.joints]),
            "mass": np.array([i.mass for i in m.inertias]),
            "com": np.array([i.com for i in m.inertias]),
            "icom": np.array([i.inertia_about_com for i in m.inertias]),
            "gravity": np.array(m.gravity),
            "q": q, "qd": qd, "u": u,
        }
        outs = {k: [] for k in ("ID.tau_out", "Minv.minv_out", "FD.qdd_out",
                                "gradID.dq_out", "gradID.dqd_out",
                                "gradFD.dq_out", "gradFD.dqd_out", "gradFD.qdd_out")}
        for k in range(N_KNOTS):
            outs["ID.tau_out"].append(refdyn.rnea(m, q[k], qd[k], u[k]))
            outs["Minv.minv_out"].append(refdyn.minv_direct(m, q[k]).ravel())
            outs["FD.qdd_out"].append(refdyn.forward_dynamics(m, q[k], qd[k], u[k]))
            g = refdyn.rnea_grad(m, q[k], qd[k], u[k])
            outs["gradID.dq_out"].append(g.dq.ravel())
            outs["gradID.dqd_out"].append(g.dqd.ravel())
            g = refdyn.fd_grad(m, q[k], qd[k], u[k])
            outs["gradFD.dq_out"].append(g.dq.ravel())
            outs["gradFD.dqd_out"].append(g.dqd.ravel())
            outs["gradFD.qdd_out"].append(refdyn.forward_dynamics(m, q[k], qd[k], u[k]))
        fx = np.random.default_rng(2).uniform(-1.0, 1.0, size=(N_KNOTS, n, 6))
        rec["f_ext"] = fx
        for k in range(N_KNOTS):
            outs.setdefault("fext.ID.tau_out", []).append(refdyn.rnea(m, q[k], qd[k], u[k], fx[k]))
            outs.setdefault("fext.FD.qdd_out", []).append(refdyn.forward_dynamics(m, q[k], qd[k], u[k], fx[k]))
            g = refdyn.rnea_grad(m, q[k], qd[k], u[k], fx[k])
            outs.setdefault("fext.gradID.dq_out", []).append(g.dq.ravel())
            outs.setdefault("fext.gradID.dqd_out", []).append(g.dqd.ravel())
            g = refdyn.fd_grad(m, q[k], qd[k], u[k], fx[k])
            outs.setdefault("fext.gradFD.dq_out", []).append(g.dq.ravel())
            outs.setdefault("fext.gradFD.dqd_out", []).append(g.dqd.ravel())
            outs.setdefault("fext.gradFD.qdd_out", []).append(refdyn.forward_dynamics(m, q[k], qd[k], u[k], fx[k]))
        for key, v in outs.items():
            rec[key] = np.array(v)
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **rec)
        print(name, n, os.path.getsize(path))


def kernel_dumps():
    """The reference's own generated programs as "rbdkernel v1" text
    (ir.py:161), written exactly as its dump_text emits them (numpy >= 2
    constants included: `np.float64(...)`)."""
    from rbdgen import codegen, ir
    for name, alg in (("chain7", "gradFD"), ("quad12", "gradID"), ("tree7", "FD"), ("mixed5", "Minv")):
        prog = codegen.build(models.load(name), alg)[0]
        path = os.path.join(HERE, f"rbdkernel_{name}_{alg}.txt")
        with open(path, "w") as fh:
            fh.write(ir.dump_text(prog))
        print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
    kernel_dumps()
