"""Topology analysis (reference `rbdgen/schedule.py:34-139`).

`build_levels` gives the depth levels the reference runs its sweeps by; the
B200 kernels evaluate a whole knot per thread, so levels no longer set the
kernel's phase structure, but they are kept for API parity and reporting.
`analyze_sparsity` names the structurally non-zero (frame, column) pairs;
the generator gets the same sparsity implicitly by folding zeros
(`codegen._Emit.lin`), and tests check both agree.
"""

from dataclasses import dataclass, field

ALGORITHMS = ("ID", "Minv", "FD", "gradID", "gradFD")


@dataclass
class LevelSchedule:
    levels: list
    level_of: list

    @property
    def depth(self):
        return len(self.levels)


def build_levels(model):
    """Frames grouped by tree depth (reference `schedule.py:44-55`)."""
    level_of = []
    for i in range(model.n_frames):
        p = model.parent[i]
        level_of.append(0 if p == -1 else level_of[p] + 1)
    levels = [[] for _ in range(max(level_of, default=-1) + 1)]
    for i, lv in enumerate(level_of):
        levels[lv].append(i)
    return LevelSchedule(levels, level_of)


@dataclass
class ColumnMap:
    """Retained (frame, column) pairs per temporary class
    (reference `schedule.py:67-114`)."""
    n_frames: int
    n_dof: int
    patterns: dict = field(default_factory=dict)

    def add(self, cls, pairs):
        self.patterns[cls] = sorted(pairs)

    def pairs(self, cls):
        return self.patterns[cls]

    def count(self, cls):
        return len(self.patterns[cls])

    def cols(self, cls, frame):
        return [c for (f, c) in self.patterns[cls] if f == frame]

    def has(self, cls, frame, col):
        return (frame, col) in set(self.patterns.get(cls, ()))

    def retained_fraction(self):
        classes = [c for c in ("grad_carry", "grad_transport") if c in self.patterns]
        if not classes:
            return 1.0
        return sum(len(self.patterns[c]) for c in classes) / (self.n_frames * self.n_dof * len(classes))


def analyze_sparsity(model, algorithm):
    """Structurally non-zero pairs (reference `schedule.py:117-139`):
    grad_carry = ancestor-or-self columns, grad_transport = that plus the
    subtree, minv_response = j >= i within the same root tree."""
    if algorithm not in ALGORITHMS:
        raise ValueError(f"unknown algorithm {algorithm!r}; expected one of {ALGORITHMS}")
    n = model.n_frames
    cmap = ColumnMap(n, model.n_dof)
    anc = [set(model.ancestors(i)) | {i} for i in range(n)]
    if algorithm in ("gradID", "gradFD"):
        cmap.add("grad_carry", [(i, j) for i in range(n) for j in anc[i]])
        cmap.add("grad_transport", [(i, j) for i in range(n) for j in anc[i] | set(model.subtree(i))])
    if algorithm in ("Minv", "FD", "gradFD"):
        root = [model.root_of(i) for i in range(n)]
        cmap.add("minv_response", [(i, j) for i in range(n) for j in range(i, n) if root[i] == root[j]])
    return cmap
