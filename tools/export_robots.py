"""Export the reference's bundled stand-in robots as URDF data files.

The reference builds its test robots as URDF text in code
(`rbdgen/models.py:63-181`: chain7 ~ iiwa, quad12 ~ HyQ, humanoid30 ~ Atlas,
plus link1, pendulum2, tree7, mixed5).  `/root/reference` is absent on the GPU
box, so the texts are committed as data under
`paper_2109_06976_b200/robots/`.  Run in the build container:

    python tools/export_robots.py
"""
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from rbdgen import models  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "paper_2109_06976_b200", "robots")

if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    for name in models.names():
        with open(os.path.join(OUT, f"{name}.urdf"), "w") as fh:
            fh.write(models.urdf_text(name))
        print("wrote", name)
