"""Boundary types and validation mirror the reference (core.py:23-190, kernels.py:36-44,366-368).

When the reference package is importable (the build container), the same inputs are fed to
both and the raised exception types / accepted cases must agree.
"""

import os
import sys

import numpy as np
import pytest

import paper_2002_03258_b200 as tsm
from conftest import REFERENCE_SRC, import_reference
from paper_2002_03258_b200.core import check_dims, validate_params_for


def test_matrix_layout_and_freeze():
    M = tsm.Matrix.from_2d([[1.0, 2.0], [3.0, 4.0], [5.0, 6.0]], tsm.Precision.DOUBLE)
    assert M.rows == 3 and M.cols == 2
    assert list(M.storage) == [1, 3, 5, 2, 4, 6]  # i + j*rows
    assert M.get(2, 1) == 6.0
    assert not M.storage.flags.writeable
    M2 = M.with_element(0, 0, 9.0)
    assert M.get(0, 0) == 1.0 and M2.get(0, 0) == 9.0
    assert np.array_equal(M.column(1), [2, 4, 6])
    assert M == tsm.Matrix.from_2d(M.to_2d(), "double")
    with pytest.raises(IndexError):
        M.get(3, 0)
    with pytest.raises(ValueError):
        tsm.Matrix(0, 2, [], tsm.Precision.DOUBLE)
    with pytest.raises(ValueError):
        tsm.Matrix(2, 2, [1.0], tsm.Precision.DOUBLE)
    with pytest.raises(ValueError):
        tsm.Matrix.from_2d([1.0, 2.0], "double")


def test_matrix_copies_storage():
    data = np.arange(6, dtype=np.float64)
    M = tsm.Matrix(2, 3, data, tsm.Precision.DOUBLE)
    data[0] = 99
    assert M.get(0, 0) == 0.0


def test_random_convention_matches_reference_draws():
    rng = np.random.default_rng(7)
    M = tsm.Matrix.random(5, 3, tsm.Precision.SINGLE, rng)
    expect = np.random.default_rng(7).random(15, dtype=np.float64).astype(np.float32)
    assert np.array_equal(M.storage, expect) and M.storage.dtype == np.float32


def test_precision_and_variant():
    assert tsm.Precision.parse("DOUBLE") is tsm.Precision.DOUBLE
    assert tsm.Precision.DOUBLE.bytes_per_element == 8 and tsm.Precision.SINGLE.bytes_per_element == 4
    assert tsm.Precision.SINGLE.eps == float(np.finfo(np.float32).eps)
    with pytest.raises(ValueError):
        tsm.Precision.parse("half")
    assert tsm.Variant.parse("L_OPT2") is tsm.Variant.L_OPT2
    assert [v.ordinal for v in tsm.Variant] == [0, 1, 2, 3, 4, 5]
    assert tsm.Variant.L_OPT1.is_tsm2l and not tsm.Variant.V3.is_tsm2l
    assert tsm.Variant.V2.uses_shared_tile and not tsm.Variant.V1.uses_shared_tile
    with pytest.raises(ValueError):
        tsm.Variant.parse("v9")


def test_params_invariants():
    for bad in (dict(t1=0), dict(t2=0), dict(t3=0), dict(tcf=0), dict(t1=32, t3=64)):
        with pytest.raises(ValueError):
            tsm.KernelParams(**bad)
    p = tsm.KernelParams(t1=128, t2=8, t3=4)
    p.validate_for(100, 100, 8)
    with pytest.raises(ValueError):
        p.validate_for(100, 100, 4)  # t2 > n
    with pytest.raises(ValueError):
        tsm.KernelParams(t1=48, t2=1, t3=4).validate_for(10, 10, 4)  # t1 % 32
    with pytest.raises(ValueError):
        tsm.KernelParams(t1=32, t2=1, t3=4, tcf=2).validate_for(10, 10, 4)  # tcf on TSM2R
    tsm.KernelParams(t1=32, t2=1, t3=4, tcf=2, variant=tsm.Variant.L_OPT1).validate_for(10, 10, 4)


def test_check_dims():
    D = tsm.Precision.DOUBLE
    A, B, C = tsm.Matrix.zeros(4, 3, D), tsm.Matrix.zeros(3, 2, D), tsm.Matrix.zeros(4, 2, D)
    assert check_dims(A, B, C) == (4, 3, 2)
    with pytest.raises(ValueError):
        check_dims(A, B, tsm.Matrix.zeros(4, 3, D))
    with pytest.raises(ValueError):
        check_dims(A, tsm.Matrix.zeros(3, 2, tsm.Precision.SINGLE), C)


def test_validate_problem():
    assert tsm.validate_problem(30720, 30720, 8) is tsm.ShapeClass.TSM2R
    assert tsm.validate_problem(1 << 24, 16, 16) is tsm.ShapeClass.TSM2L
    assert tsm.validate_problem(100, 100, 100) is tsm.ShapeClass.GENERAL
    with pytest.raises(ValueError):
        tsm.validate_problem(0, 1, 1)


def test_simulate_is_explicitly_out_of_scope():
    with pytest.raises(NotImplementedError):
        tsm.simulate()


def test_run_native_validates_before_device_work():
    """ValueErrors are raised synchronously before any device work (no GPU needed)."""
    D = tsm.Precision.DOUBLE
    A, B = tsm.Matrix.zeros(64, 8, D), tsm.Matrix.zeros(8, 4, D)
    with pytest.raises(ValueError):
        tsm.run_native(tsm.Variant.V3, A, B, tsm.Matrix.zeros(64, 8, D), tsm.KernelParams(t2=4))
    with pytest.raises(ValueError):
        tsm.run_native(tsm.Variant.V3, A, B, tsm.Matrix.zeros(64, 4, D), tsm.KernelParams(t2=8))
    with pytest.raises(ValueError):
        tsm.run_native(tsm.Variant.L_OPT2, A, B, tsm.Matrix.from_2d(np.ones((64, 4)), D),
                       tsm.KernelParams(t2=4, variant=tsm.Variant.L_OPT2))


@pytest.mark.skipif(not os.path.isdir(REFERENCE_SRC), reason="reference package only in the build container")
def test_validation_agrees_with_reference():
    sys.path.insert(0, REFERENCE_SRC)
    try:
        from tsgemm import core as rcore
    finally:
        sys.path.remove(REFERENCE_SRC)
    combos = []
    for t1 in (16, 32, 33, 64, 128):
        for t2 in (1, 4, 8, 9):
            for t3 in (1, 4, 64, 200):
                for tcf in (1, 2):
                    for var in ("v3", "l-opt1"):
                        combos.append((t1, t2, t3, tcf, var))
    for (t1, t2, t3, tcf, var) in combos:
        outcomes = []
        for mod in (rcore, tsm.core):
            try:
                p = mod.KernelParams(t1=t1, t2=t2, t3=t3, tcf=tcf, variant=mod.Variant.parse(var))
                p.validate_for(100, 50, 8)
                outcomes.append("ok")
            except ValueError:
                outcomes.append("ValueError")
        assert outcomes[0] == outcomes[1], (t1, t2, t3, tcf, var, outcomes)
    # reference Matrix objects are accepted by our validation
    rA = rcore.Matrix.zeros(8, 4, rcore.Precision.DOUBLE)
    rB = rcore.Matrix.zeros(4, 2, rcore.Precision.DOUBLE)
    rC = rcore.Matrix.zeros(8, 2, rcore.Precision.DOUBLE)
    assert check_dims(rA, rB, rC) == (8, 4, 2)
    validate_params_for(rcore.KernelParams(t1=32, t2=2, t3=4), 8, 4, 2)


def test_matrix_equality_with_reference_matrices():
    """Our Matrix compares equal to a reference Matrix with the same bits (duck-typed __eq__), and
    result_like hands back the caller's Matrix type without a copy."""
    from paper_2002_03258_b200.core import result_like
    ts = import_reference()
    data = np.arange(6, dtype=np.float64)
    ours = tsm.Matrix(2, 3, data, tsm.Precision.DOUBLE)
    ref = ts.Matrix(2, 3, data, ts.Precision.DOUBLE)
    assert ours == ref
    assert ours != ts.Matrix(2, 3, data + 1, ts.Precision.DOUBLE)
    assert ours != ts.Matrix(3, 2, data, ts.Precision.DOUBLE)
    assert ours != object()
    flat = np.arange(6, dtype=np.float64)
    r = result_like(ref, 2, 3, flat, tsm.Precision.DOUBLE)
    assert type(r) is ts.Matrix and r.precision is ts.Precision.DOUBLE
    assert r == ref and ref == r  # the reference's own __eq__ (isinstance) accepts it
    assert not r.storage.flags.writeable and np.shares_memory(r.storage, flat)
    o = result_like(ours, 2, 3, np.arange(6, dtype=np.float64), tsm.Precision.DOUBLE)
    assert type(o) is tsm.Matrix and o == ours


def test_leading_dimension_rejects_overlapping_columns():
    """gemm's stride check: expanded / stride-0 / overlapping column layouts raise."""
    import torch

    from paper_2002_03258_b200.kernels import _ld
    base = torch.zeros(8, 64, dtype=torch.float64).t()  # 64 x 8 column-major, ld 64
    assert _ld(base, 64) == 64
    assert _ld(base[:40], 40) == 64  # row sub-view keeps the parent's ld
    col = torch.zeros(64, 1, dtype=torch.float64)
    assert _ld(col, 64) == 64  # one column: stride unused
    expanded = torch.zeros(64, 1, dtype=torch.float64).expand(64, 8)  # stride (1, 0)
    with pytest.raises(ValueError):
        _ld(expanded, 64)
    overlap = torch.zeros(200, dtype=torch.float64).as_strided((64, 4), (1, 16))
    with pytest.raises(ValueError):
        _ld(overlap, 64)
    with pytest.raises(ValueError):
        _ld(torch.zeros(64, 8, dtype=torch.float64), 64)  # row-major


@pytest.mark.filterwarnings("ignore:This process .* is multi-threaded:DeprecationWarning")
def test_zero_c_scan_on_the_host_pool_and_after_fork():
    """The L_OPT2 zero-C rule on a C large enough for the library's parallel host scan (its
    persistent worker pool): ValueError with no device work, also in a forked child, which must
    not wait for the parent's workers."""
    D = tsm.Precision.DOUBLE
    m, k, n = 1 << 17, 16, 16  # 16 MB of C: several scan threads
    A, B = tsm.Matrix.zeros(m, k, D), tsm.Matrix.zeros(k, n, D)
    Cv = np.zeros((m, n))
    Cv[m - 1, n - 1] = 1.0  # the only nonzero, in the last thread's share
    C = tsm.Matrix.from_2d(Cv, D)
    p = tsm.KernelParams(t2=4, variant=tsm.Variant.L_OPT2)
    for _ in range(3):
        with pytest.raises(ValueError):
            tsm.run_native(tsm.Variant.L_OPT2, A, B, C, p)
    pid = os.fork()
    if pid == 0:  # child: same check, exit code 0 iff ValueError
        code = 1
        try:
            tsm.run_native(tsm.Variant.L_OPT2, A, B, C, p)
        except ValueError:
            code = 0
        except BaseException:
            code = 2
        os._exit(code)
    import time
    deadline = time.time() + 60
    while time.time() < deadline:
        done, status = os.waitpid(pid, os.WNOHANG)
        if done:
            assert os.WIFEXITED(status) and os.WEXITSTATUS(status) == 0, status
            return
        time.sleep(0.05)
    os.kill(pid, 9)
    os.waitpid(pid, 0)
    raise AssertionError("forked child hung in the host scan")
