"""The spec's bench_cli surface: report (pure CSV), the
kernel/schedule dumps (generation only) on CPU; validate and bench on the GPU."""
import csv
import os

import pytest

from paper_2109_06976_b200 import cli


def _csv(path, rows):
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=cli.CSV_COLUMNS)
        w.writeheader()
        for r in rows:
            w.writerow(r)


def test_report_series_and_scaling(tmp_path):
    rows = []
    for alg in ("gradFD", "ID"):
        for model, k in (("chain7", 1.0), ("quad12", 2.0)):
            for N in (16, 256):
                rows.append(dict(algorithm=alg, model=model, N=N, mode="serial", workers=1,
                                 mean_us=k * N, std_us=0, reps=3, speedup=N / 4.0))
                rows.append(dict(algorithm=alg, model=model, N=N, mode="parallel", workers=1,
                                 mean_us=k * 4.0, std_us=0, reps=3, speedup=N / 4.0))
    path = tmp_path / "lat.csv"
    _csv(path, rows)
    files = cli.cmd_report(str(path), str(tmp_path / "out"))
    # 2 algorithms -> 2 series files + 1 scaling table
    assert sorted(os.path.basename(f) for f in files) == ["scaling.tsv", "series_ID.tsv", "series_gradFD.tsv"]
    lines = open(tmp_path / "out" / "scaling.tsv").read().splitlines()[1:]
    self_ratios = [float(ln.split("\t")[4]) for ln in lines if ln.split("\t")[2] == ln.split("\t")[3]]
    assert self_ratios and all(r == 1.0 for r in self_ratios)  # a robot vs itself
    series = open(tmp_path / "out" / "series_gradFD.tsv").read().splitlines()[1:]
    serial = [float(ln.split("\t")[2]) for ln in series if ln.startswith("chain7")]
    assert serial == sorted(serial)  # serial mode monotone in N
    bad = tmp_path / "bad.csv"
    bad.write_text("x,y\n1,2\n")
    with pytest.raises(ValueError):
        cli.cmd_report(str(bad), str(tmp_path / "o2"))


def test_dumps_without_gpu(capsys):
    assert cli.main(["dump-schedule", "--model", "quad12", "--alg", "gradFD", "--warps", "4"]) == 0
    out = capsys.readouterr().out
    assert "phase 0 warp 0" in out and "arena slots" in out
    assert cli.main(["dump-kernel", "--model", "pendulum2", "--alg", "ID", "--dtype", "f64"]) == 0
    out = capsys.readouterr().out
    assert "rbd__launch_ID_f64_T" in out and "fma.rn.f64" in out
    assert cli.main(["dump-kernel", "--model", "pendulum2", "--alg", "ID", "--format", "rbdkernel"]) == 0
    out = capsys.readouterr().out
    assert out.startswith("rbdkernel v1") and "output tau_out" in out


@pytest.mark.gpu
@pytest.mark.parametrize("model", ["chain7", "quad12", "mixed5"])
def test_validate_passes(model):
    rep, ok = cli.cmd_validate(cli.argparse.Namespace(urdf=None, model=model, N=32, seed=0))
    assert ok, rep
    if model == "quad12":
        assert rep["checks"]["cross_limb_blocks_zero"]["max_dev"] == 0.0


@pytest.mark.gpu
def test_bench_rows_and_io(tmp_path):
    out = tmp_path / "lat.csv"
    assert cli.main(["bench", "--model", "chain7", "--alg", "gradFD", "--N", "16", "--N", "256",
                     "--reps", "3", "--warmup", "1", "--io-sim", "--out", str(out)]) == 0
    rows = list(csv.DictReader(open(out)))
    assert len(rows) == 4  # 2 modes x 2 Ns
    for r in rows:
        assert float(r["io_us"]) > 0
    par = {int(r["N"]): float(r["mean_us"]) for r in rows if r["mode"] == "parallel"}
    ser = {int(r["N"]): float(r["mean_us"]) for r in rows if r["mode"] == "serial"}
    assert ser[256] > par[256]
