#!/usr/bin/env python
"""Benchmark: dFD knot-points/s on B200 (BASELINE.json metric).

Headline workload (BASELINE.json configs[4], the large-batch single-GPU case
of the metric): iiwa stand-in `chain7`, gradFD (dFD = -Minv dID, plus qdd),
fp64 (the reference precision), N = 1,048,576 knot points per GPU, synthetic
seeded states.  Weak scaling: every rank evaluates its own N
knots (knots are independent; no data-path collective).

  value  knots/s, kernel only: inputs resident in HBM, one launch of the
         generated batch kernel per step, CUDA events on the launch stream,
         max over ranks.  Inputs (176 MB) and outputs (880 MB) exceed the
         126 MB L2, so no flush is needed between steps.
  e2e    knots/s through the C ABI's host-buffer entry (rbd_run_host):
         pinned host inputs -> H2D -> kernel -> D2H -> pinned host outputs,
         all inside the timed region, pipelined over the session's streams.
  roofline  fp64 CUDA-core FMA roofline: achieved = reference-IR flops per
         knot (17,131 for chain7 gradFD) x N / kernel time;
         peak = fp64 FMA throughput measured in this run (rbd_peak.cu), since
         MEASURED_PEAKS.json holds only HBM and bf16-tensor peaks.
  cpu_baseline  the oracle port of the reference CPU path
         (oracle/refdyn_np.py = rbdgen.refdyn restated) on the host cores,
         bounded sample, multiprocessing pool.
  sweep  the other BASELINE configs (iiwa N=16..256 fp32/fp64 kernel-only and
         with I/O incl. the "us per N=128 batch w/ I/O" headline, HyQ N=128,
         Atlas N=256, Atlas 1M) -- reported, not the headline.

`--impl reference` times the reference's CPU implementation (the oracle port;
the Python reference cannot travel to the GPU box) on the same workload.
"""

import argparse
import json
import multiprocessing as mp
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

REF_IR_FLOPS = {  # BASELINE.md §3, counted on the reference's generated IR (FMA = 2)
    ("chain7", "ID"): 1091, ("chain7", "Minv"): 4244, ("chain7", "FD"): 5341,
    ("chain7", "gradID"): 10870, ("chain7", "gradFD"): 17131,
    ("quad12", "ID"): 1088, ("quad12", "Minv"): 3820, ("quad12", "FD"): 4760,
    ("quad12", "gradID"): 4724, ("quad12", "gradFD"): 9548,
    ("humanoid30", "ID"): 4859, ("humanoid30", "Minv"): 22076, ("humanoid30", "FD"): 27283,
    ("humanoid30", "gradID"): 57839, ("humanoid30", "gradFD"): 96220,
}
PAPER = {"chain7": "iiwa", "quad12": "HyQ", "humanoid30": "Atlas"}


def states(n, N, seed=1, dtype=np.float64):
    rng = np.random.default_rng(seed)
    q = rng.uniform(-np.pi, np.pi, size=(N, n))
    qd = rng.uniform(-1.0, 1.0, size=(N, n))
    u = rng.uniform(-1.0, 1.0, size=(N, n))
    return [x.astype(dtype) for x in (q, qd, u)]


# ---------------------------------------------------------------------------
# CPU reference path (oracle port), multiprocessing over host cores
# ---------------------------------------------------------------------------

def _cpu_worker(args):
    robot, alg, q, qd, u = args
    sys.path.insert(0, ROOT)
    from oracle import refdyn_np as R
    from paper_2109_06976_b200 import models
    m = models.load(robot)
    for k in range(q.shape[0]):
        R.evaluate(m, alg, q[k], qd[k], u[k])
    return q.shape[0]


def cpu_reference_rate(robot, alg, sample, cores):
    """knots/s of the reference CPU path on `sample` knots over `cores` processes."""
    from paper_2109_06976_b200 import models
    n = models.load(robot).n_dof
    q, qd, u = states(n, sample, seed=1)
    chunks = [(robot, alg, q[i::cores], qd[i::cores], u[i::cores]) for i in range(cores)]
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(_cpu_worker, [(robot, alg, q[:1], qd[:1], u[:1])] * cores)  # warm (imports, parse)
        t0 = time.perf_counter()
        done = sum(pool.map(_cpu_worker, chunks))
        dt = time.perf_counter() - t0
    return done / dt, dt


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class Clocks:
    """Samples SM clock and throttle reasons every 100 ms during the timed
    region, in-process through NVML (no nvidia-smi subprocess in the loop)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _one(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        try:
            mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.samples.append((sm, mask))

    def _run(self):
        while not self._stop.is_set():
            try:
                self._one()
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=10)
            try:
                self._one()  # at least one sample at the end of the timed region
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        sm = [s for s, _ in self.samples]
        reasons = sorted({name for _, m in self.samples for bit, name in self.REASONS.items() if m & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "source": "NVML, 100 ms"}


# ---------------------------------------------------------------------------
# GPU measurements
# ---------------------------------------------------------------------------

def fma_peak_tflops(torch, dtype):
    from paper_2109_06976_b200 import kernels
    lib = kernels.peak_library()
    sink = torch.empty(256, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, iters = sms * 8, 4096
    per_iter = 2 * 16
    for _ in range(3):
        lib.rbd_fma_peak(1 if dtype == "f64" else 0, blocks, iters, sink.data_ptr(), st.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(5):
        e0.record(st)
        lib.rbd_fma_peak(1 if dtype == "f64" else 0, blocks, iters, sink.data_ptr(), st.cuda_stream)
        e1.record(st)
        e1.synchronize()
        best = max(best, float(per_iter) * iters * 256 * blocks / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


def device_rate(torch, lib, robot, alg, dt, N, steps, warmup, stream):
    """Kernel-only: ms per launch (CUDA events on the launch stream)."""
    from paper_2109_06976_b200 import codegen, models, runtime
    m = models.load(robot)
    n = m.n_dof
    tdt = torch.float64 if dt == "f64" else torch.float32
    xs = [torch.from_numpy(x).to("cuda", tdt) for x in states(n, N, seed=1)]
    nin = len(codegen.INPUTS[alg])
    outs = [torch.empty((N, e), dtype=tdt, device="cuda") for _, e in codegen.outputs(alg, n)]
    ins = [x.data_ptr() for x in xs[:nin]]
    ops = [o.data_ptr() for o in outs]
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            runtime.launch(lib, alg, dt, ins, ops, N, stream.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            runtime.launch(lib, alg, dt, ins, ops, N, stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def host_rate(torch, lib, robot, alg, dt, N, steps, warmup, reps_floor=1):
    """End to end through rbd_run_host from pinned host buffers: s per step."""
    from paper_2109_06976_b200 import codegen, models, runtime
    m = models.load(robot)
    n = m.n_dof
    tdt = torch.float64 if dt == "f64" else torch.float32
    nin = len(codegen.INPUTS[alg])
    pins = [torch.from_numpy(x).to(tdt).pin_memory() for x in states(n, N, seed=1)[:nin]]
    pouts = [torch.empty((N, e), dtype=tdt).pin_memory() for _, e in codegen.outputs(alg, n)]
    ins = [p.numpy() for p in pins]
    outs = [p.numpy() for p in pouts]
    sess = runtime.session(lib, torch.cuda.current_device())
    for _ in range(warmup):
        sess.run(alg, dt, ins, outs, N)
    t0 = time.perf_counter()
    for _ in range(steps):
        sess.run(alg, dt, ins, outs, N)
    dt_s = (time.perf_counter() - t0) / steps
    es = 8 if dt == "f64" else 4
    h2d = nin * n * N * es
    d2h = sum(e for _, e in codegen.outputs(alg, n)) * N * es
    chunks = -(-N // sess.chunk)
    # the same C-ABI call timed inside the library (no Python/ctypes overhead)
    c_s = sess.bench(alg, dt, ins, outs, N, steps)
    return dt_s, h2d, d2h, chunks, c_s


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2109_06976_b200 import kernels, models

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # RBD_BENCH_SHARED_GPU=1: every rank on cuda:0 with gloo plumbing -- only
    # to exercise the multi-rank code path on a one-GPU box (not a scaling run)
    shared = os.environ.get("RBD_BENCH_SHARED_GPU") == "1"
    if world > 1:
        torch.cuda.set_device(0 if shared else local)
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)

    robot, alg, dt, N = args.robot, args.alg, args.dtype, args.n
    m = models.load(robot)
    lib = kernels.library(m)
    meta = kernels.build_meta(m)
    stream = torch.cuda.Stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    peak64 = fma_peak_tflops(torch, "f64")
    peak32 = fma_peak_tflops(torch, "f32")

    # -- headline, kernel only ---------------------------------------------------
    barrier()
    with Clocks(0 if shared else local) as clk:
        ms = device_rate(torch, lib, robot, alg, dt, N, args.steps, args.warmup, stream)
    barrier()
    ms = max_over_ranks(ms)
    value = N * world / (ms * 1e-3)

    # -- headline, end to end via the C ABI host path ------------------------------
    barrier()
    e2e_s, h2d, d2h, chunks, e2e_c = host_rate(torch, lib, robot, alg, dt, N, max(2, args.steps // 4), 1)
    barrier()
    e2e_s = max_over_ranks(e2e_s)
    e2e = N * world / e2e_s

    flops_ref = REF_IR_FLOPS.get((robot, alg))
    flops_ours = meta["flops_per_knot"].get(f"{alg}_{dt}")
    peak = peak64 if dt == "f64" else peak32
    achieved = flops_ref * N / (ms * 1e-3) / 1e12 if flops_ref else None
    es = 8 if dt == "f64" else 4
    alg_bytes = (h2d + d2h)  # compulsory HBM bytes per launch = inputs + outputs
    traffic, traffic_src = None, None
    # dram__bytes_read+write per launch of this kernel from the newest committed
    # `ncu --set full` capture (profiles/ncu_summary_r<k>.json)
    import glob
    import re
    profs = sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_summary_r*.json")),
                   key=lambda f: int(re.search(r"_r(\d+)", f).group(1)))
    for prof in reversed(profs):
        try:
            t = json.load(open(prof)).get(f"{robot}_{alg}_{dt}", {}).get("dram_bytes_per_launch")
        except Exception:
            t = None
        if t:
            traffic, traffic_src = t * N / (1 << 20), os.path.relpath(prof, ROOT)
            break

    result = {
        "metric": f"dFD knot-points/sec ({PAPER.get(robot, robot)} stand-in {robot}, {alg}, N={N}/GPU)",
        "value": value,
        "unit": "knots/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": dt,
        "data": "synthetic seeded states q~U(-pi,pi), qd,tau~U(-1,1) (SURVEY 8d, seed 1)",
        "config": {"workload": f"{robot} {alg} {dt}, N={N} knots per GPU, one batched launch per step",
                   "robot": robot, "paper_robot": PAPER.get(robot), "algorithm": alg, "knots_per_gpu": N,
                   "parallelism": f"batch-sharded x{world}, no collective",
                   "l2": "inputs+outputs per step exceed the 126 MB L2 (no flush needed)"},
        "e2e": {"value": e2e, "unit": "knots/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_s * 1e3, "path": "Python Session.run -> rbd_run_host (C ABI, pinned host buffers)",
                "c_abi_ms_per_step": e2e_c * 1e3,
                # PCIe-bound: host<->device bytes per step over the step time
                "io_gbs": (h2d + d2h) / e2e_s / 1e9},
        "roofline": {"bound": "fp64" if dt == "f64" else "fp32",
                     "bound_note": "CUDA-core FMA pipe (no tensor-core work: 6-vector / 6x6 spatial algebra "
                                   "in fp64); HBM fraction reported alongside as hbm_frac",
                     "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": (achieved / peak) if achieved else None,
                     "traffic": traffic, "traffic_source": traffic_src, "algorithmic_bytes": alg_bytes,
                     "hbm_gbs": alg_bytes / (ms * 1e-3) / 1e9,
                     "hbm_frac": alg_bytes / (ms * 1e-3) / 1e9 / _hbm_peak(),
                     "flops_per_knot_ref_ir": flops_ref, "flops_per_knot_kernel": flops_ours,
                     "hw_frac": (flops_ours * N / (ms * 1e-3) / 1e12 / peak) if flops_ours else None,
                     "peak_source": "measured in this run: rbd_peak.cu, 16 independent fp64/fp32 FMA chains "
                                    "per thread, 64 warps/SM (nominal B200 at 1965 MHz: 37.2 TF fp64, 74.4 TF "
                                    "fp32; MEASURED_PEAKS.json has no CUDA-core FP peak)",
                     "peak_fp64_tflops": peak64, "peak_fp32_tflops": peak32},
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
    }

    # -- the other BASELINE configs (rank 0 device, not part of the headline) ------
    if rank == 0 and not args.no_sweep:
        result["sweep"] = sweep(torch, stream, args)
    if rank == 0:
        if not args.no_cpu:
            cores = host_cores()
            sample = args.cpu_sample
            rate, secs = cpu_reference_rate(robot, alg, sample, cores)
            result["cpu_baseline"] = {"value": rate, "unit": "knots/s", "cores": cores, "kind": "port",
                                      "sample": f"{sample} knots of {robot} {alg} (seed 1), "
                                                f"{secs:.1f} s wall over {cores} processes",
                                      "cpu": cpu_model()}
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _hbm_peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


def sweep(torch, stream, args):
    from paper_2109_06976_b200 import kernels, models
    out = []
    reps = max(args.steps * 10, 50)

    def entry(robot, alg, dt, N, io=True, reps=reps):
        lib = kernels.library(models.load(robot))
        ms = device_rate(torch, lib, robot, alg, dt, N, reps, 5, stream)
        rec = {"robot": robot, "paper_robot": PAPER.get(robot), "alg": alg, "dtype": dt, "N": N,
               "kernel_us": ms * 1e3, "kernel_knots_per_s": N / (ms * 1e-3)}
        fl = REF_IR_FLOPS.get((robot, alg))
        if fl:
            rec["ref_ir_tflops"] = fl * N / (ms * 1e-3) / 1e12
        if io:
            s, h2d, d2h, _, c_s = host_rate(torch, lib, robot, alg, dt, N, max(5, reps // 2) if N <= 4096 else 3, 2)
            rec.update(io_us=s * 1e6, io_knots_per_s=N / s, io_c_abi_us=c_s * 1e6)
        out.append(rec)

    for dt in ("f64", "f32"):
        for N in (16, 32, 64, 128, 256):
            for alg in ("ID", "Minv", "FD", "gradID", "gradFD"):
                entry("chain7", alg, dt, N, io=(alg == "gradFD" or N == 128))
    entry("quad12", "gradFD", "f64", 128)
    entry("quad12", "gradFD", "f32", 128)
    entry("humanoid30", "gradFD", "f64", 256)
    entry("humanoid30", "gradFD", "f32", 256)
    # device-resident rollouts (rollout.py): B trajectories x H steps of gradFD + Euler, graph-replayed
    from paper_2109_06976_b200.rollout import Rollout
    for robot, B, H in (("chain7", 128, 64), ("chain7", 4096, 64), ("humanoid30", 128, 32)):
        m = models.load(robot)
        n = m.n_dof
        r = Rollout(m, B, H, 0.01, "f64", grad=True, graph=True)
        rng = np.random.default_rng(1)
        q0 = torch.from_numpy(rng.uniform(-1, 1, (B, n))).cuda()
        tau = torch.from_numpy(rng.uniform(-1, 1, (B, H, n))).cuda()
        for _ in range(3):
            r.run(q0, q0, tau)
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(10):
            r.run(q0, q0, tau)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        out.append({"robot": robot, "paper_robot": PAPER.get(robot), "alg": "rollout(gradFD+Euler)", "dtype": "f64",
                    "N": B * H, "trajectories": B, "horizon": H, "kernel_us": ms * 1e3,
                    "kernel_knots_per_s": B * H / (ms * 1e-3), "graph": True})
    for robot in ("chain7", "quad12", "humanoid30"):
        for dt in ("f64", "f32"):
            Ns = {"chain7": (65536, 262144, 1048576), "quad12": (1048576,), "humanoid30": (65536, 262144)}[robot]
            for N in Ns:
                entry(robot, "gradFD", dt, N, io=(N == Ns[-1]), reps=max(args.steps // 2, 3))
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = host_cores()
    sample = max(cores, args.cpu_sample // 4)  # per step: ~3 s of CPU work on 16 cores
    rates = []
    for _ in range(args.warmup):
        cpu_reference_rate(args.robot, args.alg, cores * 4, cores)
    for _ in range(max(1, args.steps)):
        rates.append(cpu_reference_rate(args.robot, args.alg, sample, cores)[0])
    value = statistics.median(rates)
    print(json.dumps({
        "impl": "reference",
        "metric": f"dFD knot-points/sec ({PAPER.get(args.robot, args.robot)} stand-in {args.robot}, "
                  f"{args.alg}, N={args.n}/GPU)",
        "value": value, "unit": "knots/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": len(rates), "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic seeded states (SURVEY 8d, seed 1)",
        "config": {"workload": f"{args.robot} {args.alg} f64, N={args.n} knots per GPU "
                               f"(CPU: bounded sample of {sample} knots per step)",
                   "robot": args.robot, "algorithm": args.alg, "knots_per_gpu": args.n},
        "cpu_baseline": {"value": value, "unit": "knots/s", "cores": cores, "kind": "port",
                         "sample": f"{sample} knots per step over {cores} processes", "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "knots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--robot", default="chain7")
    ap.add_argument("--alg", default="gradFD")
    ap.add_argument("--dtype", default="f64", choices=("f64", "f32"))
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--cpu-sample", type=int, default=65536,
                    help="knots per CPU-baseline sample (~10-20 s of work on a 16-core host)")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
