"""Launch one generated batch kernel a few times (for ncu captures).

    python tools/profile_kernel.py --robot chain7 --alg gradFD --dtype f64 --n 1048576 --launches 4
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_06976_b200 import codegen, kernels, models, runtime  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--robot", default="chain7")
ap.add_argument("--alg", default="gradFD")
ap.add_argument("--dtype", default="f64")
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--launches", type=int, default=4)
ap.add_argument("--launcher", default="", help="internal launcher tag (F, W, T, P0 ...); default: the dispatch")
a = ap.parse_args()
m = models.load(a.robot)
lib = kernels.library(m)
n = m.n_dof
tdt = torch.float64 if a.dtype == "f64" else torch.float32
rng = np.random.default_rng(1)
xs = [torch.from_numpy(rng.uniform(-1, 1, (a.n, n))).to("cuda", tdt) for _ in range(3)]
outs = [torch.empty((a.n, e), dtype=tdt, device="cuda") for _, e in codegen.outputs(a.alg, n)]
nin = len(codegen.INPUTS[a.alg])
ptrs = [x.data_ptr() for x in xs[:nin]]
optr = [o.data_ptr() for o in outs]
if a.launcher:
    import ctypes
    vp = ctypes.c_void_p
    f = getattr(lib, f"rbd__launch_{a.alg}_{a.dtype}_{a.launcher}")
    f.argtypes = [vp] * 7 + [ctypes.c_int64, vp]
    f.restype = ctypes.c_int
    ia = (ptrs + [0, 0, 0])[:3] + [0] + (optr + [0, 0, 0])[:3]
for _ in range(a.launches):
    if a.launcher:
        rc = f(*[vp(p) if p else None for p in ia], ctypes.c_int64(a.n), vp(torch.cuda.current_stream().cuda_stream))
        assert rc == 0, rc
    else:
        runtime.launch(lib, a.alg, a.dtype, ptrs, optr, a.n, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", a)
