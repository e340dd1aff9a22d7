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


def test_b200_catalog_entry_loads_with_reference_loader():
    """data/gpus/b200.yaml is a catalog entry the reference's own loader reads (core.py:345-399):
    load_catalog(<dir>) / get_gpu("B200", <dir>), no unknown-key warnings, profiled winners parsed."""
    import warnings

    from conftest import import_reference
    ts = import_reference()
    from tsgemm import core as rcore
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        cat = rcore.load_catalog(cli.CATALOG_DIR)
    g = cat["B200"]
    assert g.num_sms == 148 and g.mem_bandwidth == 7300 and g.peak_gflops_double == 36400
    assert g.profiled(rcore.Precision.DOUBLE).t1 == 512 and g.profiled(rcore.Precision.DOUBLE).t2_follows_n
    assert rcore.get_gpu("B200", cli.CATALOG_DIR) == g
    # the reference's model and tuner accept it
    from tsgemm.perfmodel import t2_threshold
    assert 35 < t2_threshold(g, rcore.Precision.DOUBLE) < 45  # Peak/BW*eb, the reference's 1-flop-per-FMA form
    assert ts is not None
    assert cli.B200_SPEC["energy_pj_per_flop"]["dmma"] == 4.7  # measured after the swizzled layout


def test_run_header_has_reference_counter_columns():
    from conftest import import_reference
    import_reference()
    from tsgemm import cli as rcli
    for col in rcli._RUN_HEADER:
        if col[:2] in ("A_", "B_", "C_"):
            assert col in cli.RUN_HEADER, col


def test_paper_algorithm_loads_match_reference_oracle():
    """traffic.paper_algorithm_loads restates count_expected_loads (reference oracle.py:72-124)."""
    import itertools

    from conftest import import_reference
    import_reference()
    from tsgemm import core as rcore
    from tsgemm.oracle import count_expected_loads

    from paper_2002_03258_b200 import traffic
    for v, (m, k, n), (t1, t2, t3, tcf) in itertools.product(
            list(rcore.Variant), [(1024, 512, 8), (1000, 77, 3), (4096, 16, 16)],
            [(32, 1, 1, 1), (128, 4, 4, 2), (64, 2, 8, 3)]):
        if t2 > n:
            continue
        tcf_ = tcf if v.is_tsm2l else 1
        ref = count_expected_loads(v, m, k, n, rcore.KernelParams(t1=t1, t2=t2, t3=t3, tcf=tcf_, variant=v))
        ours = traffic.paper_algorithm_loads(v.value, m, k, n, t1, t2, t3, tcf_)
        assert ours["loads"] == ref.loads and ours["stores"] == ref.stores, (v, m, k, n, t1, t2, t3, tcf_)


def test_stream_kernel_counts_a_once():
    """The production kernel's model: A's bytes once per 16-column pass, full-segment efficiency
    for 128-B-multiple columns."""
    from paper_2002_03258_b200 import traffic, tuning
    m = k = 30720
    pl = tuning.plan("double", m, k, 8)
    c = traffic.stream_kernel_counts(pl, m, k, 8, 8, c_is_zero=False)
    assert c["A"][3] == m * k * 8 and c["A"][5] == 1.0
    assert c["C"][0] == m * 8
