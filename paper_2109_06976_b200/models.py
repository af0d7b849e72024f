"""Bundled robots (reference `rbdgen/models.py`).

The reference's fabricated stand-ins, shipped as URDF data files exported by
`tools/export_robots.py`: `chain7` (iiwa-like 7-dof chain), `quad12`
(HyQ-like 4x3 legs), `humanoid30` (Atlas-like 30-dof tree), plus `link1`,
`pendulum2`, `tree7` (paper Fig. 2 topology) and `mixed5` (prismatic and
off-axis joints).
"""

import os

from . import urdf

_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "robots")

# name -> the paper robot it stands in for (BASELINE.json configs)
PAPER_NAMES = {"chain7": "iiwa", "quad12": "HyQ", "humanoid30": "Atlas"}
BUNDLED = ("link1", "pendulum2", "chain7", "quad12", "humanoid30")


def names():
    return tuple(sorted(f[:-5] for f in os.listdir(_DIR) if f.endswith(".urdf")))


def urdf_text(name):
    path = os.path.join(_DIR, f"{name}.urdf")
    if not os.path.exists(path):
        raise KeyError(f"unknown bundled model {name!r}; available: {', '.join(names())}")
    with open(path, "r", encoding="utf-8") as fh:
        return fh.read()


def load(name, gravity=urdf.DEFAULT_GRAVITY):
    """Parse a bundled robot (reference `models.py:184`)."""
    return urdf.parse_urdf(urdf_text(name), gravity=gravity)
