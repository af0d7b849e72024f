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
a = ap.parse_args()
m = models.load(a.robot)
lib = kernels.library(m)
n = m.n_dof
tdt = torch.float64 if a.dtype == "f64" else torch.float32
rng = np.random.default_rng(1)
xs = [torch.from_numpy(rng.uniform(-1, 1, (a.n, n))).to("cuda", tdt) for _ in range(3)]
outs = [torch.empty((a.n, e), dtype=tdt, device="cuda") for _, e in codegen.outputs(a.alg, n)]
nin = len(codegen.INPUTS[a.alg])
for _ in range(a.launches):
    runtime.launch(lib, a.alg, a.dtype, [x.data_ptr() for x in xs[:nin]], [o.data_ptr() for o in outs], a.n,
                   torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", a)
