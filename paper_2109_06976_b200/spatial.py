"""Host-side spatial-algebra helpers (fp64 numpy).

Only the pieces the URDF front end and the CUDA code generator need at
generation time: rotations, spatial inertia assembly, the inertia congruence
used for fixed-joint fusion.  Conventions follow the reference
(`rbdgen/spatial.py`): spatial vectors are [angular; linear], a joint
transform is kept as (E, r) with E rotating parent coordinates into child
coordinates and r the child origin in parent coordinates, and the dense
motion transform is [[E, 0], [-E skew(r), E]] (`spatial.py:96-102`).

The per-knot arithmetic itself never runs here: it is emitted as CUDA by
`codegen.py` with every constant below baked in.
"""

import numpy as np


def skew(v):
    """3x3 matrix with skew(v) @ w == cross(v, w) (reference `spatial.py:13`)."""
    x, y, z = (float(t) for t in v)
    return np.array([[0.0, -z, y], [z, 0.0, -x], [-y, x, 0.0]])


def axis_rotation(axis, angle):
    """Right-handed Rodrigues rotation by `angle` about unit `axis`
    (reference `spatial.py:22-27`)."""
    k = skew(axis)
    return np.eye(3) + np.sin(angle) * k + (1.0 - np.cos(angle)) * (k @ k)


def rpy_matrix(roll, pitch, yaw):
    """URDF fixed-axis rpy: Rz(yaw) Ry(pitch) Rx(roll) (reference `spatial.py:30-34`)."""
    return (axis_rotation((0.0, 0.0, 1.0), yaw)
            @ axis_rotation((0.0, 1.0, 0.0), pitch)
            @ axis_rotation((1.0, 0.0, 0.0), roll))


def spatial_inertia(mass, com, icom):
    """6x6 spatial inertia about the link origin (reference `spatial.py:158-166`)."""
    c = skew(com)
    out = np.zeros((6, 6))
    out[:3, :3] = np.asarray(icom, dtype=float) + mass * (c @ c.T)
    out[:3, 3:] = mass * c
    out[3:, :3] = mass * c.T
    out[3:, 3:] = mass * np.eye(3)
    return out


def split_spatial_inertia(I):
    """(mass, com, inertia about com) of a 6x6 spatial inertia
    (reference `spatial.py:169-177`)."""
    m = I[5, 5]
    if m <= 0.0:
        return 0.0, np.zeros(3), I[:3, :3].copy()
    h = I[:3, 3:]
    com = np.array([h[2, 1], h[0, 2], h[1, 0]]) / m
    c = skew(com)
    return m, com, I[:3, :3] - m * (c @ c.T)


def joint_transform(kind, axis, origin_rotation, origin_translation, q):
    """(E, r) of a joint at position q (reference `spatial.py:180-196`)."""
    E0 = np.asarray(origin_rotation).T
    r0 = np.asarray(origin_translation, dtype=float)
    if kind == "revolute":
        return axis_rotation(axis, q).T @ E0, r0.copy()
    if kind == "prismatic":
        return E0.copy(), r0 + np.asarray(origin_rotation) @ (q * np.asarray(axis))
    if kind == "fixed":
        return E0.copy(), r0.copy()
    raise ValueError(f"unknown joint kind {kind!r}")


def motion_matrix(E, r):
    """Dense 6x6 motion transform [[E,0],[-E skew(r), E]]."""
    X = np.zeros((6, 6))
    X[:3, :3] = E
    X[3:, 3:] = E
    X[3:, :3] = -E @ skew(r)
    return X


def inertia_to_parent(E, r, I):
    """X^T I X for X = motion_matrix(E, r): an inertia in child coordinates
    re-expressed in parent coordinates (reference `spatial.py:138-155`)."""
    X = motion_matrix(E, r)
    out = X.T @ I @ X
    return 0.5 * (out + out.T)


def motion_subspace(kind, axis):
    """S = [axis; 0] for revolute, [0; axis] for prismatic (reference `spatial.py:199-206`)."""
    axis = np.asarray(axis, dtype=float)
    if kind == "revolute":
        return np.concatenate([axis, np.zeros(3)])
    if kind == "prismatic":
        return np.concatenate([np.zeros(3), axis])
    raise ValueError(f"joint kind {kind!r} has no motion subspace")
