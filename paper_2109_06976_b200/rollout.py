"""Device-resident trajectory rollouts (the paper's use case,
"tens to hundreds of naturally parallel computations ... for trajectory
optimization").

    traj = rollout(model, q0, qd0, tau, dt, grad=True)

B trajectories of H steps advance entirely on the GPU.  Default (fused):
ONE launch of `rbd_rollout` -- each CTA carries a 32-trajectory group
through the whole horizon, running the warp-specialised FD / gradFD program
and the semi-implicit Euler update (qd' = qd + dt qdd, q' = q + dt qd')
step after step with no launch in between.  fused=False keeps the per-step
form: one batched dynamics launch over the B knots (FD, or gradFD when the
per-knot Jacobians are wanted -- it returns qdd too) and one
`rbd_euler_step` per step, captured once in a CUDA graph and replayed.
States are time-major, [H+1][B][n], so every step's knots are contiguous.
No host synchronisation or copy happens inside the loop.

Semantics per step k (reference functions restated, refdyn.py:172-175 and
:242-249): qdd_k = FD(q_k, qd_k, tau_k); with grad=True also
(dqdd/dq, dqdd/dqd)_k = fd_grad(q_k, qd_k, tau_k).
"""

import ctypes

from . import kernels, runtime

_DT = {"f32": 0, "f64": 1}


class Rollout:
    """Reusable device-resident rollout for fixed (B, H, dt, dtype, grad);
    `run(q0, qd0, tau)` fills `q`, `qd` ([H+1, B, n]), `qdd` ([H, B, n]) and,
    with grad, `dq`, `dqd` ([H, B, n, n]) in place."""

    def __init__(self, model, B, H, dt, dtype="f64", grad=False, graph=True, device=None, fused=None):
        import torch
        self.torch = torch
        self.model, self.B, self.H, self.dt, self.dtype, self.grad = model, int(B), int(H), float(dt), dtype, grad
        if dtype not in _DT:
            raise ValueError(f"dtype must be 'f32' or 'f64', got {dtype!r}")
        self.lib = kernels.library(model)
        n = model.n_dof
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        tdt = torch.float64 if dtype == "f64" else torch.float32
        z = lambda *s: torch.zeros(s, dtype=tdt, device=self.device)
        self.q, self.qd = z(H + 1, B, n), z(H + 1, B, n)
        self.tau, self.qdd = z(H, B, n), z(H, B, n)
        self.dq = z(H, B, n, n) if grad else None
        self.dqd = z(H, B, n, n) if grad else None
        self._graph = None
        self._use_graph = graph
        if fused is None:  # per-robot measured choice (codegen TUNED "rollout_fused")
            from . import codegen
            fused = bool(codegen.tuning(model, "gradFD" if grad else "FD", dtype).get("rollout_fused", True))
        self.fused = fused

    def _steps(self, stream):
        lib, B, dt = self.lib, self.B, self.dtype
        for k in range(self.H):
            ins = [self.q[k].data_ptr(), self.qd[k].data_ptr(), self.tau[k].data_ptr()]
            if self.grad:
                outs = [self.dq[k].data_ptr(), self.dqd[k].data_ptr(), self.qdd[k].data_ptr()]
                runtime.launch(lib, "gradFD", dt, ins, outs, B, stream)
            else:
                runtime.launch(lib, "FD", dt, ins, [self.qdd[k].data_ptr()], B, stream)
            rc = lib.rbd_euler_step(_DT[dt], ctypes.c_void_p(self.q[k].data_ptr()),
                                    ctypes.c_void_p(self.qd[k].data_ptr()), ctypes.c_void_p(self.qdd[k].data_ptr()),
                                    ctypes.c_void_p(self.q[k + 1].data_ptr()),
                                    ctypes.c_void_p(self.qd[k + 1].data_ptr()), ctypes.c_int64(B),
                                    ctypes.c_double(self.dt), ctypes.c_void_p(stream))
            runtime.check(rc, "rbd_euler_step")

    def run(self, q0, qd0, tau):
        """q0, qd0: [B, n]; tau: [B, H, n] (CUDA tensors).  Asynchronous on
        the current stream; returns self."""
        torch = self.torch
        n = self.model.n_dof
        for nm, x, shp in (("q0", q0, (self.B, n)), ("qd0", qd0, (self.B, n)), ("tau", tau, (self.B, self.H, n))):
            if tuple(x.shape) != shp:
                raise ValueError(f"{nm} has shape {tuple(x.shape)}, expected {shp}")
        self.q[0].copy_(q0)
        self.qd[0].copy_(qd0)
        self.tau.copy_(tau.transpose(0, 1))
        stream = torch.cuda.current_stream(self.device)
        if self.fused:
            vp = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
            rc = self.lib.rbd_rollout(4 if self.grad else 2, _DT[self.dtype], vp(self.q), vp(self.qd), vp(self.tau),
                                      vp(self.qdd), vp(self.dq), vp(self.dqd), ctypes.c_int64(self.B),
                                      ctypes.c_int32(self.H), ctypes.c_double(self.dt),
                                      ctypes.c_void_p(stream.cuda_stream))
            runtime.check(rc, "rbd_rollout")
            return self
        if not self._use_graph:
            self._steps(stream.cuda_stream)
            return self
        if self._graph is None:
            # warm up (lazy per-device caches, smem opt-in) outside the capture
            side = torch.cuda.Stream(self.device)
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                self._steps(side.cuda_stream)
            stream.wait_stream(side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._steps(torch.cuda.current_stream(self.device).cuda_stream)
            self._graph = g
        self._graph.replay()
        return self

    def trajectories(self):
        """(q, qd, qdd[, dq, dqd]) batch-major: [B, H+1, n], [B, H+1, n], [B, H, n], [B, H, n, n] x 2."""
        out = [self.q.transpose(0, 1), self.qd.transpose(0, 1), self.qdd.transpose(0, 1)]
        if self.grad:
            out += [self.dq.transpose(0, 1), self.dqd.transpose(0, 1)]
        return tuple(out)


def rollout(model, q0, qd0, tau, dt, grad=False, graph=False, fused=None):
    """One-shot rollout of B = q0.shape[0] trajectories over H = tau.shape[1]
    steps (CUDA tensors); returns `Rollout.trajectories()`."""
    dtype = "f32" if q0.dtype == __import__("torch").float32 else "f64"
    r = Rollout(model, q0.shape[0], tau.shape[1], dt, dtype, grad, graph, fused=fused)
    return r.run(q0, qd0, tau).trajectories()


__all__ = ["Rollout", "rollout"]
