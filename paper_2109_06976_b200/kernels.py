"""Build and load the generated per-robot sm_100a libraries.

`library(model)` returns the loaded C-ABI library (`include/rbd_b200.h`) for
a robot, compiling it first when no build for the model's fingerprint exists.
Builds live IN-TREE under `paper_2109_06976_b200/_build/<robot>-<hash>/` so
they travel to the GPU box with the repo snapshot; `__graft_entry__.build()`
prebuilds every bundled robot.

There is no fallback: if the library cannot be built or loaded, or no CUDA
device is present when a kernel is launched, the call raises.
"""

import concurrent.futures as cf
import ctypes
import json
import os
import re
import shutil
import subprocess
import threading

from . import codegen

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(os.path.dirname(PKG), "include")
BUILD = os.environ.get("RBD_B200_BUILD_DIR", os.path.join(PKG, "_build"))

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH_FLAGS + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                           "-Xptxas", "-v", "-diag-suppress", "177", "-I", CSRC, "-I", INCLUDE]


class BuildError(RuntimeError):
    pass


def _nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise BuildError("nvcc not found: the generated sm_100a kernels cannot be built")


def build_dir(model):
    # RBD_BUILD_KEY: a fixed key for tuning experiments (tools/variants.sh), so
    # an experiment build stays addressable while the generator keeps changing
    key = os.environ.get("RBD_BUILD_KEY") or codegen.tuning_key()
    return os.path.join(BUILD, f"{model.name}-{codegen.model_hash(model)[:16]}-{key}")


def library_path(model):
    return os.path.join(build_dir(model), f"librbd_{model.name}.so")


def _parse_ptxas(log):
    """{kernel symbol: {registers, spill_stores, spill_loads, stack}} from -Xptxas -v."""
    out, cur = {}, None
    for line in log.splitlines():
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
            out[cur] = {}
            continue
        if cur is None:
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and "stack" not in out[cur]:
            out[cur].update(stack=int(m.group(1)), spill_stores=int(m.group(2)), spill_loads=int(m.group(3)))
        m = re.search(r"Used (\d+) registers", line)
        if m:
            out[cur]["registers"] = int(m.group(1))
    return out


def compile_library(model, force=False, jobs=None, algorithms=codegen.ALGORITHMS, dtypes=codegen.DTYPES):
    """Generate + compile the robot's library; returns the .so path."""
    path = library_path(model)
    if os.path.exists(path) and not force:
        return path
    nvcc = _nvcc()
    bdir = build_dir(model)
    tmp = bdir + ".tmp%d" % os.getpid()
    shutil.rmtree(tmp, ignore_errors=True)
    os.makedirs(tmp)
    files, flops = codegen.generate_sources(model, algorithms, dtypes)
    for name, text in files.items():
        with open(os.path.join(tmp, name), "w") as fh:
            fh.write(text)
    units = sorted(f for f in files if f.endswith(".cu"))
    # biggest translation units first
    units.sort(key=lambda f: -len(files[f]))

    def one(unit):
        obj = os.path.join(tmp, unit[:-3] + ".o")
        cmd = [nvcc] + NVCC_FLAGS + ["-I", tmp, "-c", os.path.join(tmp, unit), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise BuildError(f"nvcc failed on {unit}:\n{r.stderr[-4000:]}")
        return obj, r.stderr

    jobs = jobs or max(1, min(len(units), os.cpu_count() or 1))
    with cf.ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(one, units))
    objs = [o for o, _ in results]
    log = "\n".join(l for _, l in results)
    so = os.path.join(tmp, os.path.basename(path))
    r = subprocess.run([nvcc] + ARCH_FLAGS + ["-shared", "-o", so] + objs, capture_output=True, text=True)
    if r.returncode != 0:
        raise BuildError(f"link failed:\n{r.stderr[-4000:]}")
    with open(os.path.join(tmp, "ptxas.log"), "w") as fh:
        fh.write(log)
    meta = {
        "robot": model.name,
        "fingerprint": codegen.model_hash(model),
        "n_dof": model.n_dof,
        "flops_per_knot": {f"{a}_{d}": v for (a, d), v in flops.items()},
        "ptxas": _parse_ptxas(log),
        "nvcc_flags": NVCC_FLAGS,
        "tuning_env": os.environ.get("RBD_TUNING", ""),  # non-empty: an experiment build (tools/variants.sh)
    }
    with open(os.path.join(tmp, "meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    keep_src = os.environ.get("RBD_KEEP_SOURCES") == "1"  # generated .cu kept for inspection only on request
    for f in os.listdir(tmp):
        if f.endswith(".o") or (not keep_src and f.startswith("k_") and f.endswith(".cu")):
            os.remove(os.path.join(tmp, f))
    shutil.rmtree(bdir, ignore_errors=True)
    os.replace(tmp, bdir)
    return path


def build_meta(model):
    with open(os.path.join(build_dir(model), "meta.json")) as fh:
        return json.load(fh)


# ---------------------------------------------------------------------------
# ctypes binding of include/rbd_b200.h
# ---------------------------------------------------------------------------

class RbdInfo(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_int32), ("n_dof", ctypes.c_int32),
                ("n_frames", ctypes.c_int32), ("n_trees", ctypes.c_int32),
                ("knots_per_block", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("robot", ctypes.c_char_p), ("fingerprint", ctypes.c_char_p)]


ABI_SYMBOLS = (["rbd_get_info", "rbd_alg_extents", "rbd_launch", "rbd_launch_fext", "rbd_session_create",
                "rbd_session_destroy", "rbd_run_host", "rbd_run_host_fext", "rbd_bench_host",
                "rbd_run_host_multi", "rbd_run_host_multi_fext", "rbd_session_device",
                "rbd_euler_step", "rbd_rollout"]
               + [f"rbd_{a}_{d}" for a in codegen.ALGORITHMS for d in codegen.DTYPES]
               + [f"rbd_{a}_{d}_fext" for a in codegen.FEXT_ALGORITHMS for d in codegen.DTYPES])

_vp = ctypes.c_void_p


def _bind(lib):
    lib.rbd_get_info.argtypes = [ctypes.POINTER(RbdInfo)]
    lib.rbd_alg_extents.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int32)] + [ctypes.POINTER(ctypes.c_int64)] * 3
    lib.rbd_launch.argtypes = [ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int64, _vp]
    lib.rbd_launch_fext.argtypes = [ctypes.c_int, ctypes.c_int] + [_vp] * 7 + [ctypes.c_int64, _vp]
    lib.rbd_euler_step.argtypes = [ctypes.c_int] + [_vp] * 5 + [ctypes.c_int64, ctypes.c_double, _vp]
    if hasattr(lib, "rbd_rollout") or os.environ.get("RBD_PARTIAL_BUILD") != "1":
        lib.rbd_rollout.argtypes = [ctypes.c_int, ctypes.c_int] + [_vp] * 6 + [ctypes.c_int64, ctypes.c_int32,
                                                                                ctypes.c_double, _vp]
    lib.rbd_run_host_fext.argtypes = [_vp, ctypes.c_int, ctypes.c_int] + [_vp] * 7 + [ctypes.c_int64]
    lib.rbd_session_create.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(_vp)]
    lib.rbd_session_destroy.argtypes = [_vp]
    lib.rbd_session_device.argtypes = [_vp, ctypes.POINTER(ctypes.c_int32)]
    lib.rbd_run_host_multi.argtypes = [ctypes.POINTER(_vp), ctypes.c_int32, ctypes.c_int, ctypes.c_int] + [_vp] * 6 \
        + [ctypes.c_int64]
    lib.rbd_run_host_multi_fext.argtypes = [ctypes.POINTER(_vp), ctypes.c_int32, ctypes.c_int, ctypes.c_int] \
        + [_vp] * 7 + [ctypes.c_int64]
    lib.rbd_run_host.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int64]
    lib.rbd_bench_host.argtypes = ([_vp, ctypes.c_int, ctypes.c_int] + [_vp] * 6
                                   + [ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_double)])
    for a in codegen.ALGORITHMS:
        for d in codegen.DTYPES:
            try:
                fn = getattr(lib, f"rbd_{a}_{d}")
            except AttributeError:
                if os.environ.get("RBD_PARTIAL_BUILD") == "1":  # experiment builds of a few entries
                    continue
                raise
            fn.argtypes = [_vp] * 6 + [ctypes.c_int64, _vp]
            fn.restype = ctypes.c_int
            if a in codegen.FEXT_ALGORITHMS:
                getattr(lib, f"rbd_{a}_{d}_fext").argtypes = [_vp] * 7 + [ctypes.c_int64, _vp]
                getattr(lib, f"rbd_{a}_{d}_fext").restype = ctypes.c_int
    for s in ABI_SYMBOLS:
        if not hasattr(lib, s) and os.environ.get("RBD_PARTIAL_BUILD") == "1":
            continue
        getattr(lib, s).restype = ctypes.c_int
    return lib


_LOCK = threading.Lock()
_LIBS = {}


def load_library(path):
    return _bind(ctypes.CDLL(path))


def library(model, build=True):
    """Loaded ctypes library for `model` (compiling it if needed)."""
    key = codegen.model_hash(model)
    with _LOCK:
        lib = _LIBS.get((key, codegen.tuning_key()))
        if lib is None:
            path = library_path(model)
            if not os.path.exists(path):
                if not build:
                    raise BuildError(f"no prebuilt library for {model.name!r} at {path}")
                compile_library(model)
            lib = load_library(path)
            info = RbdInfo()
            if lib.rbd_get_info(ctypes.byref(info)) != 0 or info.fingerprint.decode() != key:
                raise BuildError(f"library at {path} does not match model {model.name!r}")
            _LIBS[(key, codegen.tuning_key())] = lib
        return lib


def peak_library(force=False):
    """librbd_peak.so: the CUDA-core FMA roofline probe (csrc/rbd_peak.cu)."""
    out = os.path.join(BUILD, "librbd_peak.so")
    if force or not os.path.exists(out):
        os.makedirs(BUILD, exist_ok=True)
        r = subprocess.run([_nvcc()] + ARCH_FLAGS + ["-O3", "-shared", "-Xcompiler", "-fPIC", "-o", out + ".tmp",
                            os.path.join(CSRC, "rbd_peak.cu")], capture_output=True, text=True)
        if r.returncode != 0:
            raise BuildError(r.stderr[-4000:])
        os.replace(out + ".tmp", out)
    lib = ctypes.CDLL(out)
    lib.rbd_fma_peak.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    lib.rbd_fma_peak.restype = ctypes.c_int
    return lib
