"""Compare two dump_outputs.py files bit for bit (NaN = never written)."""
import sys

import numpy as np

a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
bad = 0
for k in sorted(a.files):
    x, y = a[k], b[k]
    same = np.array_equal(x.view(np.uint8), y.view(np.uint8))
    print(k, x.shape, "identical" if same else f"DIFFER max {np.nanmax(np.abs(x - y)):.3e}",
          "nan" if np.isnan(y).any() else "")
    bad += (not same) or np.isnan(y).any()
sys.exit(1 if bad else 0)
