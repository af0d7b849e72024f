"""Small-batch latency probe: per-launch device time of each kernel mapping
of a robot's library (the internal launchers rbd__launch_<alg>_<dt>_<tag>),
from a CUDA graph of back-to-back launches (no host launch overhead in the
number), at several batch sizes.  Usage:
  python tools/small_n.py chain7 [algs] [dtypes] [Ns]"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_06976_b200 import codegen, kernels, models  # noqa: E402


def graph_time(fn, reps=50, rounds=5):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            fn(st.cuda_stream)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                fn(st.cuda_stream)
        g.replay()
        st.synchronize()
        best = None
        for _ in range(rounds):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.replay()
            e1.record(st)
            e1.synchronize()
            t = e0.elapsed_time(e1) * 1e3 / reps
            best = t if best is None else min(best, t)
    return best


def main():
    robot = sys.argv[1] if len(sys.argv) > 1 else "chain7"
    algs = sys.argv[2].split(",") if len(sys.argv) > 2 else list(codegen.ALGORITHMS)
    dts = sys.argv[3].split(",") if len(sys.argv) > 3 else ["f64", "f32"]
    Ns = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [16, 128, 256, 1024, 4096]
    m = models.load(robot)
    lib = kernels.library(m)
    n = m.n_dof
    vp = ctypes.c_void_p
    for alg in algs:
        for dt in dts:
            tdt = torch.float64 if dt == "f64" else torch.float32
            for N in Ns:
                rng = np.random.default_rng(1)
                xs = [torch.from_numpy(rng.uniform(-1, 1, (N, n))).to("cuda", tdt) for _ in range(3)]
                outs = [torch.empty((N, e), dtype=tdt, device="cuda") for _, e in codegen.outputs(alg, n)]
                ptr = [x.data_ptr() for x in xs] + [0] + [o.data_ptr() for o in outs] + [0] * (3 - len(outs))
                rec = {"robot": robot, "alg": alg, "dtype": dt, "N": N}
                for tag in ("S", "C", "F", "W", "T", ""):
                    name = f"rbd__launch_{alg}_{dt}_{tag}" if tag else f"rbd__launch_{alg}_{dt}"
                    try:
                        f = getattr(lib, name)
                    except AttributeError:
                        continue
                    f.argtypes = [vp] * 7 + [ctypes.c_int64, vp]
                    f.restype = ctypes.c_int

                    def fn(s, f=f):
                        rc = f(*[vp(p) if p else None for p in ptr], ctypes.c_int64(N), vp(s))
                        assert rc == 0, rc
                    rec[tag or "dispatch"] = round(graph_time(fn), 2)
                print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
