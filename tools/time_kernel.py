"""Time one generated kernel (CUDA events), print a JSON line.  Honors RBD_TUNING.

    RBD_TUNING='{"bk":128}' python tools/time_kernel.py --robot chain7 --alg gradFD --dtype f64 --n 1048576
"""
import argparse
import json
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
ap.add_argument("--n", type=int, nargs="+", default=[1 << 20])
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
m = models.load(a.robot)
lib = kernels.library(m)
meta = kernels.build_meta(m)
n = m.n_dof
tdt = torch.float64 if a.dtype == "f64" else torch.float32
for N in a.n:
    rng = np.random.default_rng(1)
    xs = [torch.from_numpy(rng.uniform(-1, 1, (N, n))).to("cuda", tdt) for _ in range(3)]
    outs = [torch.empty((N, e), dtype=tdt, device="cuda") for _, e in codegen.outputs(a.alg, n)]
    nin = len(codegen.INPUTS[a.alg])
    st = torch.cuda.current_stream()
    args = ([x.data_ptr() for x in xs[:nin]], [o.data_ptr() for o in outs], N, st.cuda_stream)
    for _ in range(3):
        runtime.launch(lib, a.alg, a.dtype, *args)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.reps):
        runtime.launch(lib, a.alg, a.dtype, *args)
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / a.reps
    ptx = {k: v for k, v in meta["ptxas"].items() if f"Knot_{a.alg}_{a.dtype}" in k}
    print(json.dumps({"tuning": os.environ.get("RBD_TUNING", ""), "robot": a.robot, "alg": a.alg, "dtype": a.dtype,
                      "N": N, "us": us, "knots_per_s": N / us * 1e6, "ptxas": list(ptx.values())}), flush=True)
