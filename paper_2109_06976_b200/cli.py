"""Command-line harness mirroring the reference spec's `bench_cli` / `batch_exec`
surface: ``validate``, ``bench``, ``report``,
``dump-kernel``, ``dump-schedule``.

    python -m paper_2109_06976_b200.cli validate --model chain7
    python -m paper_2109_06976_b200.cli bench --model chain7 --alg gradFD --N 16 --N 256 --out lat.csv
    python -m paper_2109_06976_b200.cli report lat.csv --out series/
    python -m paper_2109_06976_b200.cli dump-kernel --model chain7 --alg gradFD --dtype f64
    python -m paper_2109_06976_b200.cli dump-schedule --model humanoid30 --alg gradFD

Everything runs through the product path (the generated sm_100a kernels via
the C ABI); `validate` checks the kernels against themselves (central finite
differences of FD/ID, FD∘ID round trips, Minv symmetry/positivity,
cross-limb zero blocks) -- the reference-equivalence suite lives in tests/.

Modes of `bench` (the spec's batch_exec modes, on the GPU):
  serial    N launches of one knot each, back to back (the reference's
            one-knot-per-call interpreter loop)
  parallel  one batched launch of N knots (GRiD's one block per computation)
CSV columns {algorithm, model, N, mode, workers, mean_us, std_us, reps}
 plus `speedup` (serial_mean / parallel_mean) and, with
--io-sim, `io_us` (host buffers through rbd_run_host: H2D + kernel + D2H).
"""

import argparse
import csv
import json
import os
import statistics
import sys
import time

import numpy as np

from . import codegen, dynamics, kernels, models, runtime, urdf

CSV_COLUMNS = ["algorithm", "model", "N", "mode", "workers", "mean_us", "std_us", "reps", "speedup"]


def _load_model(args):
    if getattr(args, "urdf", None):
        return urdf.parse_urdf(args.urdf)
    return models.load(args.model)


def _states(n, N, seed):
    rng = np.random.default_rng(seed)
    return (rng.uniform(-np.pi, np.pi, (N, n)), rng.uniform(-1, 1, (N, n)), rng.uniform(-1, 1, (N, n)))


# ---------------------------------------------------------------------------
# validate
# ---------------------------------------------------------------------------

def cmd_validate(args):
    """Self-consistency of the generated kernels (SPEC.md:505-514 structure).
    Returns (report dict, ok)."""
    m = _load_model(args)
    n = m.n_dof
    q, qd, u = _states(n, args.N, args.seed)
    rep = {"model": m.name, "n_dof": n, "N": args.N, "checks": {}}
    ok = True

    def record(name, value, tol):
        nonlocal ok
        passed = bool(value <= tol)
        ok &= passed
        rep["checks"][name] = {"max_dev": float(value), "tol": tol, "pass": passed}

    # FD o ID round trip and ID o FD (SPEC acceptance 3)
    qdd = dynamics.forward_dynamics(m, q, qd, u)
    tau = dynamics.rnea(m, q, qd, qdd)
    record("FD_then_ID", float(np.max(np.abs(tau - u)) / max(1.0, np.max(np.abs(u)))), 1e-8)
    Minv = dynamics.minv_direct(m, q)
    record("Minv_symmetric", float(np.max(np.abs(Minv - np.swapaxes(Minv, 1, 2)))), 1e-10)
    ev = np.linalg.eigvalsh(0.5 * (Minv + np.swapaxes(Minv, 1, 2)))
    record("Minv_positive_definite", float(max(0.0, -ev.min())), 0.0)
    # FD = Minv (tau - c) consistency between the Minv and FD kernels
    c = dynamics.bias_force(m, q, qd)
    fd2 = np.einsum("kij,kj->ki", Minv, u - c)
    record("FD_equals_Minv_tau_minus_c", float(np.max(np.abs(fd2 - qdd)) / max(1.0, np.max(np.abs(qdd)))), 1e-9)
    # analytical gradients vs central finite differences of the kernels (SPEC acceptance 2)
    h = 1e-6
    k = min(args.N, 8)
    g_id = dynamics.rnea_grad(m, q[:k], qd[:k], qdd[:k])
    g_fd = dynamics.fd_grad(m, q[:k], qd[:k], u[:k])
    worst_id = worst_fd = 0.0
    for j in range(n):
        e = np.zeros(n)
        e[j] = h
        for which, (g, fn, x3) in {"ID": (g_id, dynamics.rnea, qdd[:k]),
                                   "FD": (g_fd, dynamics.forward_dynamics, u[:k])}.items():
            dq_fd = (fn(m, q[:k] + e, qd[:k], x3) - fn(m, q[:k] - e, qd[:k], x3)) / (2 * h)
            dqd_fd = (fn(m, q[:k], qd[:k] + e, x3) - fn(m, q[:k], qd[:k] - e, x3)) / (2 * h)
            for an, num in ((g.dq[:, :, j], dq_fd), (g.dqd[:, :, j], dqd_fd)):
                dev = float(np.max(np.abs(an - num) / (1e-7 / 1e-5 + np.abs(num))))
                if which == "ID":
                    worst_id = max(worst_id, dev)
                else:
                    worst_fd = max(worst_fd, dev)
    record("gradID_vs_finite_differences", worst_id, 1e-5)
    record("gradFD_vs_finite_differences", worst_fd, 1e-5)
    # branch independence: cross-limb blocks exactly 0
    roots = [m.root_of(i) for i in range(n)]
    mask = np.array([[roots[i] != roots[j] for j in range(n)] for i in range(n)])
    if mask.any():
        cross = max(float(np.max(np.abs(g_fd.dq[:, mask]))), float(np.max(np.abs(g_fd.dqd[:, mask]))),
                    float(np.max(np.abs(Minv[:, mask]))))
        record("cross_limb_blocks_zero", cross, 0.0)
    rep["coverage"] = {"algorithms": list(codegen.ALGORITHMS), "dtypes": ["f64"]}
    return rep, ok


# ---------------------------------------------------------------------------
# bench (batch_exec.sweep on the GPU)
# ---------------------------------------------------------------------------

def _time_device(torch, lib, alg, dt, xs, outs, N, reps, warmup, one_by_one):
    st = torch.cuda.current_stream()
    nin = len(codegen.INPUTS[alg])

    def once():
        if one_by_one:
            for k in range(N):
                runtime.launch(lib, alg, dt, [x[k:k + 1].data_ptr() for x in xs[:nin]],
                               [o[k:k + 1].data_ptr() for o in outs], 1, st.cuda_stream)
        else:
            runtime.launch(lib, alg, dt, [x.data_ptr() for x in xs[:nin]], [o.data_ptr() for o in outs], N,
                           st.cuda_stream)

    for _ in range(warmup):
        once()
    torch.cuda.synchronize()
    samples = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        once()
        e1.record(st)
        e1.synchronize()
        samples.append(e0.elapsed_time(e1) * 1e3)
    return samples


def cmd_bench(args):
    """Latency table rows (dicts, CSV_COLUMNS order) for every algorithm x N."""
    import torch
    m = _load_model(args)
    lib = kernels.library(m)
    n = m.n_dof
    dt = args.dtype
    tdt = torch.float64 if dt == "f64" else torch.float32
    rows = []
    for alg in args.alg:
        for N in args.N:
            q, qd, u = _states(n, N, args.seed)
            xs = [torch.from_numpy(x).to("cuda", tdt) for x in (q, qd, u)]
            outs = [torch.empty((N, e), dtype=tdt, device="cuda") for _, e in codegen.outputs(alg, n)]
            means = {}
            for mode in ("serial", "parallel"):
                s = _time_device(torch, lib, alg, dt, xs, outs, N, args.reps, args.warmup, mode == "serial")
                means[mode] = statistics.mean(s)
                rows.append({"algorithm": alg, "model": m.name, "N": N, "mode": mode, "workers": 1,
                             "mean_us": statistics.mean(s), "std_us": statistics.pstdev(s), "reps": len(s)})
            for r in rows[-2:]:
                r["speedup"] = means["serial"] / means["parallel"]
            if args.io_sim:
                ndt = np.float64 if dt == "f64" else np.float32
                hin = [torch.from_numpy(x.astype(ndt)).pin_memory().numpy() for x in (q, qd, u)]
                hout = [torch.empty((N, e), dtype=tdt).pin_memory().numpy() for _, e in codegen.outputs(alg, n)]
                sess = runtime.session(lib, torch.cuda.current_device())
                nin = len(codegen.INPUTS[alg])
                sess.run(alg, dt, hin[:nin], hout, N)
                sec = sess.bench(alg, dt, hin[:nin], hout, N, args.reps)
                for r in rows[-2:]:
                    r["io_us"] = sec * 1e6
    return rows


def write_csv(rows, path):
    cols = CSV_COLUMNS + (["io_us"] if rows and "io_us" in rows[0] else [])
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=cols)
        w.writeheader()
        for r in rows:
            w.writerow({c: r.get(c) for c in cols})


# ---------------------------------------------------------------------------
# report
# ---------------------------------------------------------------------------

def cmd_report(csv_path, out_dir):
    """Per-algorithm series files (N vs mean latency per mode, N vs speedup)
    and a scaling table across robots.  Returns the list of
    files written."""
    try:
        with open(csv_path) as fh:
            rows = list(csv.DictReader(fh))
        for r in rows:
            r["N"] = int(r["N"])
            r["mean_us"] = float(r["mean_us"])
    except (KeyError, ValueError) as e:
        raise ValueError(f"malformed CSV {csv_path}: {e}") from e
    os.makedirs(out_dir, exist_ok=True)
    written = []
    algs = sorted({r["algorithm"] for r in rows})
    for alg in algs:
        path = os.path.join(out_dir, f"series_{alg}.tsv")
        with open(path, "w") as fh:
            fh.write("model\tN\tserial_mean_us\tparallel_mean_us\tspeedup\n")
            for model in sorted({r["model"] for r in rows if r["algorithm"] == alg}):
                for N in sorted({r["N"] for r in rows if r["algorithm"] == alg and r["model"] == model}):
                    sel = {r["mode"]: r["mean_us"] for r in rows
                           if r["algorithm"] == alg and r["model"] == model and r["N"] == N}
                    s, p = sel.get("serial"), sel.get("parallel")
                    fh.write(f"{model}\t{N}\t{s}\t{p}\t{(s / p) if s and p else ''}\n")
        written.append(path)
    # scaling table: model A parallel latency / model B parallel latency per algorithm (Fig. 4)
    path = os.path.join(out_dir, "scaling.tsv")
    mods = sorted({r["model"] for r in rows})
    with open(path, "w") as fh:
        fh.write("algorithm\tN\tmodel_a\tmodel_b\tratio\n")
        for alg in algs:
            for N in sorted({r["N"] for r in rows if r["algorithm"] == alg}):
                par = {r["model"]: r["mean_us"] for r in rows
                       if r["algorithm"] == alg and r["N"] == N and r["mode"] == "parallel"}
                for a in mods:
                    for b in mods:
                        if a in par and b in par:
                            fh.write(f"{alg}\t{N}\t{a}\t{b}\t{par[a] / par[b]}\n")
    written.append(path)
    return written


# ---------------------------------------------------------------------------
# dumps
# ---------------------------------------------------------------------------

def cmd_dump_kernel(args):
    """The generated CUDA translation unit(s) of one (robot, algorithm, dtype),
    or (--format rbdkernel) the program in the reference's kernel text format."""
    m = _load_model(args)
    if getattr(args, "format", "cuda") == "rbdkernel":
        from . import kdump
        return kdump.dump_text(m, args.alg, args.dtype)
    files, _ = codegen.generate_sources(m, algorithms=(args.alg,), dtypes=(args.dtype,))
    return "\n".join(f"// ===== {nm}\n{txt}" for nm, txt in sorted(files.items()) if nm != "main.cu")


def cmd_dump_schedule(args):
    """The warp-specialised schedule: phases, per-warp tasks, arena slots."""
    from . import wsched
    m = _load_model(args)
    P = wsched.plan(m, args.alg, args.dtype, args.warps)
    S = P["sched"]
    lines = [f"# {m.name} {args.alg} {args.dtype}: {len(S.task_ops)} tasks, {len(S.phases)} phases, "
             f"{args.warps} warps, {S.nslots} arena slots, critical path {S.critical_path()} of {S.total()} ops"]
    for p, ph in enumerate(S.phases):
        for w, tasks in enumerate(ph):
            if tasks:
                lines.append(f"phase {p} warp {w}: " + " ".join(f"{t}({S.cost[t]})" for t in tasks))
    return "\n".join(lines)


# ---------------------------------------------------------------------------

def main(argv=None):
    ap = argparse.ArgumentParser(prog="paper_2109_06976_b200.cli", description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="verb", required=True)

    def common(p, alg_multi=False):
        p.add_argument("--urdf", help="URDF file or XML text (default: --model)")
        p.add_argument("--model", default="chain7", help="bundled model name")
        p.add_argument("--dtype", default="f64", choices=codegen.DTYPES)
        p.add_argument("--seed", type=int, default=0)
        if alg_multi:
            p.add_argument("--alg", action="append", choices=codegen.ALGORITHMS)
        else:
            p.add_argument("--alg", default="gradFD", choices=codegen.ALGORITHMS)

    p = sub.add_parser("validate")
    common(p)
    p.add_argument("--N", type=int, default=64)
    p.add_argument("--out")
    p = sub.add_parser("bench")
    common(p, alg_multi=True)
    p.add_argument("--N", type=int, action="append")
    p.add_argument("--workers", type=int, default=1)
    p.add_argument("--reps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--io-sim", action="store_true")
    p.add_argument("--out", default="latency.csv")
    p = sub.add_parser("report")
    p.add_argument("csv")
    p.add_argument("--out", default="report")
    p = sub.add_parser("dump-kernel")
    common(p)
    p.add_argument("--format", choices=("cuda", "rbdkernel"), default="cuda")
    p = sub.add_parser("dump-schedule")
    common(p)
    p.add_argument("--warps", type=int, default=8)
    args = ap.parse_args(argv)

    if args.verb == "validate":
        rep, ok = cmd_validate(args)
        text = json.dumps(rep, indent=1)
        if args.out:
            with open(args.out, "w") as fh:
                fh.write(text)
        print(text)
        return 0 if ok else 1
    if args.verb == "bench":
        args.alg = args.alg or ["gradFD"]
        args.N = args.N or [16, 32, 64, 128, 256]
        if args.workers != 1:
            print("note: --workers has no effect on the GPU executor (one launch per batch)", file=sys.stderr)
        t0 = time.time()
        rows = cmd_bench(args)
        write_csv(rows, args.out)
        print(f"wrote {len(rows)} rows to {args.out} in {time.time() - t0:.1f} s")
        return 0
    if args.verb == "report":
        for f in cmd_report(args.csv, args.out):
            print(f)
        return 0
    if args.verb == "dump-kernel":
        print(cmd_dump_kernel(args))
        return 0
    if args.verb == "dump-schedule":
        print(cmd_dump_schedule(args))
        return 0
    return 2


if __name__ == "__main__":
    sys.exit(main())
