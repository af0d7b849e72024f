import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
MODELS = ("link1", "pendulum2", "chain7", "quad12", "humanoid30", "tree7", "mixed5")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long CPU-side build (skipped unless RBD_SLOW=1)")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("RBD_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow build test; set RBD_SLOW=1")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)


def golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def rel_err(y, ref):
    """Per-knot norm-wise relative error: max|y-ref| / max|ref|."""
    y = np.asarray(y, dtype=np.float64).reshape(len(ref), -1)
    ref = np.asarray(ref, dtype=np.float64).reshape(len(ref), -1)
    num = np.max(np.abs(y - ref), axis=1)
    den = np.maximum(np.max(np.abs(ref), axis=1), 1e-300)
    return float(np.max(num / den))


# tolerances stated by the north star (BASELINE.json): fp64 1e-9 relative,
# fp32 1e-4 relative against fp64 evaluation of the fp32-rounded inputs
TOL = {"f64": 1e-9, "f32": 1e-4}
