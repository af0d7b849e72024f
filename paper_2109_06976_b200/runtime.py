"""Thin Python side of the C ABI (`include/rbd_b200.h`).

Launches go through the per-robot library's `rbd_<alg>_<dt>` (device
pointers, caller's stream) or `rbd_run_host` (host buffers, the library's own
pipelined session).  Nothing here computes dynamics; a failing launch raises.
"""

import ctypes
import threading

from . import codegen, kernels

_ALG_ID = {a: i for i, a in enumerate(codegen.ALGORITHMS)}
_DT_ID = {"f32": 0, "f64": 1}

_CUDA_ERRORS = {
    1: "cudaErrorInvalidValue", 2: "cudaErrorMemoryAllocation", 3: "cudaErrorInitializationError",
    35: "cudaErrorInsufficientDriver", 100: "cudaErrorNoDevice", 101: "cudaErrorInvalidDevice",
    209: "cudaErrorNoKernelImageForDevice", 400: "cudaErrorInvalidResourceHandle",
    700: "cudaErrorIllegalAddress", 701: "cudaErrorLaunchOutOfResources",
}


class LaunchError(RuntimeError):
    pass


def check(rc, what):
    if rc == 0:
        return
    if rc < 0:
        raise ValueError(f"{what}: invalid argument (rbd error {rc})")
    name = _CUDA_ERRORS.get(rc, "cudaError")
    hint = ""
    if rc in (35, 100, 209):
        hint = " -- the generated kernels need a CUDA B200 (sm_100a); there is no CPU fallback"
    raise LaunchError(f"{what}: {name} ({rc}){hint}")


def robot_library(model):
    return kernels.library(model)


def launch(lib, alg, dtype, in_ptrs, out_ptrs, N, stream, fext_ptr=None):
    """One batched kernel launch on device pointers (asynchronous); with
    fext_ptr, the f_ext entry rbd_<alg>_<dt>_fext."""
    ins = list(in_ptrs) + [None] * (3 - len(in_ptrs))
    outs = list(out_ptrs) + [None] * (3 - len(out_ptrs))
    vp = lambda p: ctypes.c_void_p(p) if p else None
    st = ctypes.c_void_p(stream) if stream else None
    if fext_ptr is not None:
        name = f"rbd_{alg}_{dtype}_fext"
        rc = getattr(lib, name)(*[vp(p) for p in ins], vp(fext_ptr), *[vp(p) for p in outs],
                                ctypes.c_int64(N), st)
    else:
        name = f"rbd_{alg}_{dtype}"
        rc = getattr(lib, name)(*[vp(p) for p in ins + outs], ctypes.c_int64(N), st)
    check(rc, name)


class Session:
    """Owns an `rbd_session` (device buffers + streams for the host path)."""

    def __init__(self, lib, device=0, chunk_knots=65536, slots=3):
        self.lib = lib
        self.device = device
        self.chunk = int(chunk_knots)
        h = ctypes.c_void_p()
        check(lib.rbd_session_create(int(device), ctypes.c_int64(self.chunk), int(slots), ctypes.byref(h)),
              "rbd_session_create")
        self.handle = h

    def run(self, alg, dtype, in_arrays, out_arrays, N, f_ext=None):
        ins = [a.ctypes.data_as(ctypes.c_void_p) for a in in_arrays] + [None] * (3 - len(in_arrays))
        outs = [a.ctypes.data_as(ctypes.c_void_p) for a in out_arrays] + [None] * (3 - len(out_arrays))
        if f_ext is not None:
            rc = self.lib.rbd_run_host_fext(self.handle, _ALG_ID[alg], _DT_ID[dtype], *ins,
                                            f_ext.ctypes.data_as(ctypes.c_void_p), *outs, ctypes.c_int64(N))
            check(rc, f"rbd_run_host_fext({alg}, {dtype})")
            return
        rc = self.lib.rbd_run_host(self.handle, _ALG_ID[alg], _DT_ID[dtype], *ins, *outs, ctypes.c_int64(N))
        check(rc, f"rbd_run_host({alg}, {dtype})")

    def bench(self, alg, dtype, in_arrays, out_arrays, N, reps):
        """Mean wall seconds per rbd_run_host call, timed inside the library
        (rbd_bench_host: the latency a C/C++ caller sees)."""
        ins = [a.ctypes.data_as(ctypes.c_void_p) for a in in_arrays] + [None] * (3 - len(in_arrays))
        outs = [a.ctypes.data_as(ctypes.c_void_p) for a in out_arrays] + [None] * (3 - len(out_arrays))
        sec = ctypes.c_double()
        rc = self.lib.rbd_bench_host(self.handle, _ALG_ID[alg], _DT_ID[dtype], *ins, *outs, ctypes.c_int64(N),
                                     int(reps), ctypes.byref(sec))
        check(rc, f"rbd_bench_host({alg}, {dtype})")
        return sec.value

    def close(self):
        if self.handle:
            self.lib.rbd_session_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_SESS_LOCK = threading.Lock()
_SESSIONS = {}


def default_chunk(lib):
    """~64 MiB of fp64 per pipeline stage."""
    worst = 0
    for a in range(5):
        ni, e0, e1, e2 = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        lib.rbd_alg_extents(a, ctypes.byref(ni), ctypes.byref(e0), ctypes.byref(e1), ctypes.byref(e2))
        info = kernels.RbdInfo()
        lib.rbd_get_info(ctypes.byref(info))
        worst = max(worst, ni.value * info.n_dof + e0.value + e1.value + e2.value)
    return max(4096, min(1 << 20, (64 << 20) // (8 * max(worst, 1))))


def session(lib, device=0):
    key = (id(lib), device)
    with _SESS_LOCK:
        s = _SESSIONS.get(key)
        if s is None:
            s = Session(lib, device, default_chunk(lib))
            _SESSIONS[key] = s
        return s


def run_host(lib, alg, dtype, in_arrays, out_arrays, N, device=None, f_ext=None):
    session(lib, 0 if device is None else device).run(alg, dtype, in_arrays, out_arrays, N, f_ext)
