"""The GPU-backed experiment front-end (paper_2002_03258_b200.cli): CSV conventions on CPU, and
measured rows on the GPU."""

import csv

import pytest

from paper_2002_03258_b200 import cli
from paper_2002_03258_b200.core import Precision


def _read(path):
    with open(path, newline="") as fh:
        return list(csv.reader(fh))


def test_model_table(tmp_path):
    out = str(tmp_path / "model.csv")
    assert cli.main(["model", "--out", out]) == 0
    rows = _read(out)
    assert rows[0] == cli.MODEL_HEADER
    bounds = {int(r[7]): r[12] for r in rows[1:]}
    assert bounds[2] == bounds[8] == bounds[16] == "memory"  # every BASELINE config is HBM-bound
    ridge = float(rows[1][2])
    assert 16 < ridge < 24
    # the power-cap bound: above the memory bound, growing with n
    pred = [float(r[15]) for r in rows[1:]]
    assert all(float(r[15]) >= float(r[10]) for r in rows[1:]) and pred == sorted(pred)
    assert rows[3][13] == "dmma" and rows[1][13] == "dfma"
    assert open(out, "rb").read().count(b"\r") == 0


def test_unknown_gpu_and_header_only(tmp_path):
    assert cli.main(["model", "--gpu", "K40c", "--out", str(tmp_path / "x.csv")]) == 2
    out = str(tmp_path / "run.csv")
    # no variants -> header-only CSV, as the reference (test_cli.py:40-49); no GPU needed
    assert cli.cmd_run(Precision.DOUBLE, [(64, 64, 4)], [], {}, 0, out) == 0
    assert _read(out) == [cli.RUN_HEADER]


def test_atomic_write_leaves_no_partial_file(tmp_path):
    out = tmp_path / "bad.csv"

    def rows():
        yield [1, 2]
        raise RuntimeError("boom")
    with pytest.raises(RuntimeError):
        cli._write_csv(str(out), ["a", "b"], rows())
    assert not out.exists() and not list(tmp_path.glob("*.tmp"))


@pytest.mark.gpu
def test_run_measured_rows(tmp_path):
    out = str(tmp_path / "run.csv")
    assert cli.main(["run", "--m", "4096", "--k", "4096", "--n", "8", "--variant", "v3", "--variant", "v1",
                     "--variant", "v2", "--out", out, "--reps", "3"]) == 0
    rows = _read(out)
    h = rows[0]
    for r in rows[1:]:
        d = dict(zip(h, r))
        assert d["error"] == ""
        assert float(d["time_ms"]) > 0 and float(d["check_rel_frobenius"]) <= 1e-12
    # infeasible params surface as a per-row error (reference test_cli.py:68-82)
    out2 = str(tmp_path / "bad.csv")
    assert cli.main(["run", "--m", "256", "--k", "256", "--n", "4", "--variant", "v3", "--t1", "33",
                     "--out", out2]) == 0
    d = dict(zip(*_read(out2)))
    assert "ValueError" in d["error"]
