"""Run one generated entry on seeded inputs and save its outputs (.npz), so
two tuning variants of the same program can be compared bit for bit.

    RBD_PARTIAL_BUILD=1 RBD_TUNING='{...}' RBD_BUILD_KEY=x... \\
        python tools/experiments/dump_outputs.py chain7 gradFD f64 out.npz 1000 65541
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_06976_b200 import codegen, kernels, models, runtime  # noqa: E402

robot, alg, dt, path = sys.argv[1:5]
m = models.load(robot)
lib = kernels.library(m)
n = m.n_dof
tdt = torch.float64 if dt == "f64" else torch.float32
res = {}
for N in map(int, sys.argv[5:]):
    rng = np.random.default_rng(N)
    xs = [torch.from_numpy(rng.uniform(-1, 1, (N, n))).to("cuda", tdt) for _ in range(3)]
    outs = [torch.full((N, e), float("nan"), dtype=tdt, device="cuda") for _, e in codegen.outputs(alg, n)]
    nin = len(codegen.INPUTS[alg])
    runtime.launch(lib, alg, dt, [x.data_ptr() for x in xs[:nin]], [o.data_ptr() for o in outs], N,
                   torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for k, o in enumerate(outs):
        res[f"{N}_{k}"] = o.cpu().numpy()
np.savez(path, **res)
print("saved", path, sorted(res))
