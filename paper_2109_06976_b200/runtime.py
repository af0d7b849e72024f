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
    if rc == -3:  # RBD_ENONFINITE (refdyn._check_state)
        raise ValueError("state vector contains non-finite entries")
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
        ins = [a.ctypes.data for a in in_arrays] + [None] * (3 - len(in_arrays))
        outs = [a.ctypes.data for a in out_arrays] + [None] * (3 - len(out_arrays))
        if f_ext is not None:
            rc = self.lib.rbd_run_host_fext(self.handle, _ALG_ID[alg], _DT_ID[dtype], *ins,
                                            f_ext.ctypes.data, *outs, N)
            check(rc, f"rbd_run_host_fext({alg}, {dtype})")
            return
        rc = self.lib.rbd_run_host(self.handle, _ALG_ID[alg], _DT_ID[dtype], *ins, *outs, N)
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
    info = kernels.RbdInfo()
    lib.rbd_get_info(ctypes.byref(info))
    for a in range(5):
        ni, e0, e1, e2 = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        lib.rbd_alg_extents(a, ctypes.byref(ni), ctypes.byref(e0), ctypes.byref(e1), ctypes.byref(e2))
        worst = max(worst, ni.value * info.n_dof + e0.value + e1.value + e2.value)
    return max(4096, min(1 << 20, (64 << 20) // (8 * max(worst, 1))))


def current_device():
    """The caller's current CUDA device (torch's, when torch is in use), else 0."""
    import sys
    torch = sys.modules.get("torch")
    if torch is not None:
        try:
            if torch.cuda.is_initialized():
                return torch.cuda.current_device()
        except Exception:
            pass
    return 0


def session(lib, device=None, lane=0):
    """The calling host thread's session on `device` (default: the current
    device).  Sessions own pinned staging and device buffers, so each host
    thread gets its own (the C ABI's rule: a session is not shared between
    threads); `lane` tells apart the sessions of one multi-device call (a
    device may appear twice in its list).  They live as long as the library."""
    dev = current_device() if device is None else int(device)
    key = (id(lib), dev, threading.get_ident(), lane)
    with _SESS_LOCK:
        s = _SESSIONS.get(key)
        if s is None:
            s = Session(lib, dev, default_chunk(lib))
            _SESSIONS[key] = s
        return s


def shard_ranges(N, count):
    """Contiguous slices [(begin, length)] of ceil(N / count) knots -- the
    split rbd_run_host_multi makes (rbd_runtime.cuh rbd_shard)."""
    per = -(-int(N) // int(count)) if count > 0 else 0
    out = []
    for k in range(count):
        b = min(per * k, N)
        out.append((b, min(b + per, N) - b))
    return out


def run_host(lib, alg, dtype, in_arrays, out_arrays, N, device=None, f_ext=None, devices=None):
    """Host buffers through the library's pipeline.  devices=[d0, d1, ...]:
    the batch is sliced across those GPUs (rbd_run_host_multi: one session
    and host thread per device, slices run concurrently)."""
    if not devices or len(devices) == 1:
        dev = devices[0] if devices else device
        session(lib, dev).run(alg, dtype, in_arrays, out_arrays, N, f_ext)
        return
    sess = [session(lib, d, lane=1 + k) for k, d in enumerate(devices)]
    arr = (ctypes.c_void_p * len(sess))(*[s.handle.value for s in sess])
    ins = [a.ctypes.data_as(ctypes.c_void_p) for a in in_arrays] + [None] * (3 - len(in_arrays))
    outs = [a.ctypes.data_as(ctypes.c_void_p) for a in out_arrays] + [None] * (3 - len(out_arrays))
    if f_ext is not None:
        rc = lib.rbd_run_host_multi_fext(arr, len(sess), _ALG_ID[alg], _DT_ID[dtype], *ins,
                                         f_ext.ctypes.data_as(ctypes.c_void_p), *outs, ctypes.c_int64(N))
    else:
        rc = lib.rbd_run_host_multi(arr, len(sess), _ALG_ID[alg], _DT_ID[dtype], *ins, *outs, ctypes.c_int64(N))
    check(rc, f"rbd_run_host_multi({alg}, {dtype}, {len(sess)} devices)")
