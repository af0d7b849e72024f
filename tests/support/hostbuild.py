"""TEST-ONLY: host (g++) build of the generated per-knot programs.

The generator emits plain C++ for the one-knot program (knots_<alg>_<dt>.h);
compiling it for the host lets the CPU test tier check the generator against
the oracle without a GPU.  Never used by the product API.
"""
import ctypes
import os
import subprocess

import numpy as np

from paper_2109_06976_b200 import codegen, kernels

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "_hostbuild")


def host_library(model, opt="-O0"):
    d = os.path.join(OUT, f"{model.name}-{codegen.model_hash(model)[:16]}-{codegen.tuning_key()}")
    so = os.path.join(d, "host.so")
    if not os.path.exists(so):
        os.makedirs(d, exist_ok=True)
        for nm, txt in codegen.host_sources(model).items():
            with open(os.path.join(d, nm), "w") as fh:
                fh.write(txt)
        cmd = ["g++", opt, "-std=c++17", "-x", "c++", "-I", kernels.CSRC, "-I", kernels.INCLUDE,
               "-I", d, '-DGEN_SRC="host_all.h"', "-shared", "-fPIC", "-o", so + ".tmp",
               os.path.join(HERE, "host_harness.cpp")]
        subprocess.run(cmd, check=True, capture_output=True)
        os.replace(so + ".tmp", so)
    lib = ctypes.CDLL(so)
    lib.host_eval.argtypes = [ctypes.c_int, ctypes.c_int] + [ctypes.c_void_p] * 6 + [ctypes.c_int64]
    lib.host_eval_fext.argtypes = [ctypes.c_int, ctypes.c_int] + [ctypes.c_void_p] * 7 + [ctypes.c_int64]
    return lib


def host_eval(lib, model, alg, dtype, q, qd, u, f_ext=None):
    ndt = np.float64 if dtype == "f64" else np.float32
    arrs = [np.ascontiguousarray(x, dtype=ndt) for x in (q, qd, u)]
    N = arrs[0].shape[0]
    outs = [np.zeros((N, e), ndt) for _, e in codegen.outputs(alg, model.n_dof)]
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    optrs = [ptr(o) for o in outs] + [None] * (3 - len(outs))
    if f_ext is not None:
        fx = np.ascontiguousarray(f_ext, dtype=ndt).reshape(N, -1)
        rc = lib.host_eval_fext(codegen.ALGORITHMS.index(alg), codegen.DTYPES.index(dtype),
                                *[ptr(a) for a in arrs], ptr(fx), *optrs, N)
        assert rc == 0
        return {nm: o for (nm, _), o in zip(codegen.outputs(alg, model.n_dof), outs)}
    rc = lib.host_eval(codegen.ALGORITHMS.index(alg), codegen.DTYPES.index(dtype),
                       *[ptr(a) for a in arrs], *optrs, N)
    assert rc == 0
    return {nm: o for (nm, _), o in zip(codegen.outputs(alg, model.n_dof), outs)}
