"""Batched drop-in for the reference dynamics API (`rbdgen/refdyn.py:91-249`).

Same names, argument order and error behaviour as the reference, evaluated
by the generated sm_100a kernels:

    rnea(model, q, qd, qdd)              -> tau
    bias_force(model, q, qd)             -> c = rnea(q, qd, 0)
    minv_direct(model, q)                -> Minv
    forward_dynamics(model, q, qd, tau)  -> qdd
    rnea_grad(model, q, qd, qdd)         -> DynamicsGradients(dq, dqd)
    fd_grad(model, q, qd, tau)           -> DynamicsGradients(dq, dqd) (+ .qdd)

State arguments may be one knot `(n,)` (the reference's literal signature)
or a batch `(N, n)`:

* numpy arrays / sequences run through the host-buffer path of the C ABI
  (`rbd_run_host`: chunked H2D -> kernel -> D2H pipeline) and return numpy;
* CUDA torch tensors run through the device path (`rbd_<alg>_<dt>` on the
  current torch stream, no copies, no synchronisation) and return CUDA
  tensors.

float32 inputs select the fp32 kernels, everything else fp64 (the reference
precision); `dtype="f32"|"f64"` overrides.  Shapes other than (n,) / (N, n)
raise ValueError as `refdyn._check_state` does (`refdyn.py:31-38`); host
inputs containing non-finite values raise ValueError too (checked by the C
ABI's host path: on the host for small batches, on the device per staged
chunk for large ones).  `f_ext` (per-link
external forces in link coordinates, refdyn.py:79-80) is `(n, 6)` for one
knot or `(N, n, 6)`, and runs the f_ext kernels (`rbd_<alg>_<dt>_fext`; the
reference's generated programs have no f_ext input, its refdyn does).
`devices=[0, 1, ...]` slices a host batch across several GPUs (contiguous
ceil(N / G) slices, one session and host thread per GPU, results in place;
knots are independent, so there is no exchange step).
"""

from dataclasses import dataclass

import numpy as np

from . import codegen, runtime

_ALG_ID = {a: i for i, a in enumerate(codegen.ALGORITHMS)}


@dataclass
class DynamicsGradients:
    """Partials of a joint-space output w.r.t. q (dq) and qd (dqd)
    (reference `refdyn.py:23-28`); fd_grad also carries the solved qdd."""
    dq: object
    dqd: object
    qdd: object = None


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _resolve_dtype(arrs, dtype):
    if dtype is not None:
        if dtype not in ("f32", "f64"):
            raise ValueError(f"dtype must be 'f32' or 'f64', got {dtype!r}")
        return dtype
    x = arrs[0]
    if _is_torch(x):
        import torch
        return "f32" if x.dtype == torch.float32 else "f64"
    return "f32" if getattr(np.asarray(x), "dtype", None) == np.float32 else "f64"


def _shape_check(model, arrs):
    n = model.n_dof
    single = None
    N = None
    for x in arrs:
        shp = tuple(x.shape)
        if len(shp) == 1 and shp[0] == n:
            s, k = True, 1
        elif len(shp) == 2 and shp[1] == n:
            s, k = False, shp[0]
        else:
            raise ValueError(f"state vector has shape {shp}, expected ({n},) or (N, {n})")
        if single is None:
            single, N = s, k
        elif s != single or k != N:
            raise ValueError("state arguments disagree in batch shape")
    return single, N


def _fext_shape(model, fx, single, N):
    n = model.n_dof
    shp = tuple(fx.shape)
    want = (n, 6) if single else (N, n, 6)
    if shp != want:
        raise ValueError(f"f_ext has shape {shp}, expected {want}")


_PIN_BYTES = 1 << 20  # host outputs at least this large come from the pinned pool


def _host_empty(shape, ndt):
    """Output array for the host path.  Large outputs are page-locked, taken
    from torch's caching pinned-host allocator (blocks return to the pool
    when the array is freed), so the D2H copies run at full PCIe speed
    instead of through pageable staging."""
    nbytes = shape[0] * shape[1] * (8 if ndt == np.float64 else 4)
    if nbytes >= _PIN_BYTES:
        try:
            import torch
            if torch.cuda.is_available():
                tdt = torch.float32 if ndt == np.float32 else torch.float64
                return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()
        except Exception:
            pass
    return np.empty(shape, dtype=ndt)


_NDOF = {}


def _ndof(model):
    """model.n_dof, memoised per model object (the property walks the joints)."""
    ent = _NDOF.get(id(model))
    if ent is not None and ent[0] is model:
        return ent[1]
    n = model.n_dof
    _NDOF[id(model)] = (model, n)
    return n


def _host_fast(model, alg, args):
    """The common host call -- C-contiguous float64/float32 numpy arrays of
    one shape, no f_ext / device options -- with the checks done once
    (same results and errors as the general path, fewer Python steps)."""
    x0 = args[0]
    if type(x0) is not np.ndarray:
        return None
    ndt, shp = x0.dtype, x0.shape
    if ndt != np.float64 and ndt != np.float32:
        return None
    for x in args:
        if type(x) is not np.ndarray or x.dtype != ndt or x.shape != shp or not x.flags.c_contiguous:
            return None
    n = _ndof(model)
    if len(shp) == 2 and shp[1] == n:
        single, N = False, shp[0]
    elif len(shp) == 1 and shp[0] == n:
        single, N = True, 1
    else:
        return None  # the general path raises the reference's error
    # non-finite inputs: rejected by the host path itself (RBD_ENONFINITE ->
    # ValueError, refdyn._check_state), checked on the device for big batches
    dt = "f32" if ndt == np.float32 else "f64"
    outs_spec = codegen.outputs(alg, n)
    outs = [_host_empty((N, e), ndt) for _, e in outs_spec]
    runtime.run_host(runtime.robot_library(model), alg, dt, args, outs, N)
    return [o.reshape((n, n) if e == n * n else (n,)) if single else
            o.reshape((N, n, n) if e == n * n else (N, n)) for (_, e), o in zip(outs_spec, outs)]


def _run(model, alg, args, dtype=None, device=None, f_ext=None, devices=None):
    """Evaluate `alg` on state arguments `args` (1 or 3 arrays), optionally
    with per-link external forces f_ext; host arrays may be sliced across
    several GPUs (`devices`)."""
    if dtype is None and device is None and f_ext is None and devices is None:
        fast = _host_fast(model, alg, args)
        if fast is not None:
            return fast
    dt = _resolve_dtype(args, dtype)
    on_device = _is_torch(args[0]) and args[0].is_cuda
    lib = runtime.robot_library(model)
    n = model.n_dof
    if on_device:
        import torch
        tdt = torch.float32 if dt == "f32" else torch.float64
        dev = args[0].device
        xs = []
        for x in args:
            if not (_is_torch(x) and x.is_cuda and x.device == dev):
                raise ValueError("mixing device and host state arguments")
            xs.append(x.to(tdt).contiguous())
        single, N = _shape_check(model, xs)
        fx = None
        if f_ext is not None:
            if not (_is_torch(f_ext) and f_ext.is_cuda and f_ext.device == dev):
                raise ValueError("mixing device and host state arguments")
            fx = f_ext.to(tdt).contiguous()
            _fext_shape(model, fx, single, N)
        if devices:
            raise ValueError("devices= applies to host arrays; a CUDA tensor runs on its own device")
        outs = [torch.empty((N, e), dtype=tdt, device=dev) for _, e in codegen.outputs(alg, n)]
        with torch.cuda.device(dev):
            stream = torch.cuda.current_stream(dev).cuda_stream
            runtime.launch(lib, alg, dt, [x.data_ptr() for x in xs],
                           [o.data_ptr() for o in outs], N, stream,
                           fext_ptr=None if fx is None else fx.data_ptr())
    else:
        ndt = np.float32 if dt == "f32" else np.float64
        xs = []
        for x in args:
            if _is_torch(x):
                x = x.detach().cpu().numpy()
            xs.append(np.ascontiguousarray(np.asarray(x, dtype=ndt)))
        single, N = _shape_check(model, xs)
        fx = None
        if f_ext is not None:
            fx = f_ext.detach().cpu().numpy() if _is_torch(f_ext) else f_ext
            fx = np.ascontiguousarray(np.asarray(fx, dtype=ndt))
            _fext_shape(model, fx, single, N)
        # non-finite inputs raise ValueError from the host path (RBD_ENONFINITE)
        outs = [_host_empty((N, e), ndt) for _, e in codegen.outputs(alg, n)]
        runtime.run_host(lib, alg, dt, xs, outs, N, device=device, f_ext=fx, devices=devices)
    shaped = []
    for (nm, e), o in zip(codegen.outputs(alg, n), outs):
        shp = (n, n) if e == n * n else (n,)
        shaped.append(o.reshape(shp) if single else o.reshape((N,) + shp))
    return shaped


def rnea(model, q, qd, qdd, f_ext=None, dtype=None, devices=None):
    """Inverse dynamics (reference `refdyn.py:91-94`)."""
    return _run(model, "ID", [q, qd, qdd], dtype, f_ext=f_ext, devices=devices)[0]


def bias_force(model, q, qd, f_ext=None, dtype=None, devices=None):
    """rnea at qdd = 0 (reference `refdyn.py:97-100`)."""
    if _is_torch(q):
        import torch
        zero = torch.zeros_like(q)
    else:
        zero = np.zeros_like(np.asarray(q, dtype=np.float32 if _resolve_dtype([q], dtype) == "f32" else np.float64))
    return _run(model, "ID", [q, qd, zero], dtype, f_ext=f_ext, devices=devices)[0]


def minv_direct(model, q, dtype=None, devices=None):
    """Direct inverse mass matrix (reference `refdyn.py:128-169`)."""
    return _run(model, "Minv", [q], dtype, devices=devices)[0]


def forward_dynamics(model, q, qd, tau, f_ext=None, dtype=None, devices=None):
    """qdd = Minv (tau - c) (reference `refdyn.py:172-175`)."""
    return _run(model, "FD", [q, qd, tau], dtype, f_ext=f_ext, devices=devices)[0]


def rnea_grad(model, q, qd, qdd, f_ext=None, dtype=None, devices=None):
    """(dtau/dq, dtau/dqd) (reference `refdyn.py:178-239`)."""
    dq, dqd = _run(model, "gradID", [q, qd, qdd], dtype, f_ext=f_ext, devices=devices)
    return DynamicsGradients(dq, dqd)


def fd_grad(model, q, qd, tau, f_ext=None, dtype=None, devices=None):
    """(dqdd/dq, dqdd/dqd) = -Minv dID at qdd = FD(q, qd, tau)
    (reference `refdyn.py:242-249`); the solved qdd rides along."""
    dq, dqd, qdd = _run(model, "gradFD", [q, qd, tau], dtype, f_ext=f_ext, devices=devices)
    return DynamicsGradients(dq, dqd, qdd)
