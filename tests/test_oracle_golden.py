"""Pins the CPU oracle (oracle/reference.py) to the reference package's own outputs.

tests/golden/golden.json was produced by tests/golden/make_golden.py running the reference
(``tsgemm.kernels.run_native`` and ``tsgemm.oracle.naive_gemm``) on the reference's test inputs.
Here the inputs are regenerated with the reference's RNG conventions (digests must match), our
restatements are run, and their outputs must be BITWISE equal to the reference's.
"""

import numpy as np
import pytest

from conftest import golden, golden_cases, regenerate, sha
from oracle import max_rel_error, naive_gemm, run_native_port, run_native_port_threaded


@pytest.mark.parametrize("case", golden_cases(), ids=lambda c: c["name"])
def test_inputs_regenerate(case):
    A, B, C0 = regenerate(case)
    assert sha(A) == case["sha_A"]
    assert sha(B) == case["sha_B"]
    assert sha(C0) == case["sha_C0"]


@pytest.mark.parametrize("case", golden_cases(), ids=lambda c: c["name"])
def test_naive_gemm_bitwise(case):
    A, B, C0 = regenerate(case)
    out = naive_gemm(A, B, C0)
    assert sha(out) == case["sha_naive_gemm"]
    if case.get("arrays"):
        arr = golden()[1][case["name"] + "/naive_gemm"]
        assert np.array_equal(out.reshape(-1, order="F"), arr)


@pytest.mark.parametrize("case", golden_cases(), ids=lambda c: c["name"])
def test_run_native_port_bitwise(case):
    A, B, C0 = regenerate(case)
    out = run_native_port(A, B, C0, case["params"]["t2"])
    assert sha(out) == case["sha_run_native"]
    ref = naive_gemm(A, B, C0)
    assert max_rel_error(out, ref) == pytest.approx(case["ref_max_rel_error"], rel=0, abs=0)


def test_threaded_port_is_bitwise_single():
    rng = np.random.default_rng(1)
    A, B, C = rng.random((1001, 300)), rng.random((300, 8)), rng.random((1001, 8))
    assert np.array_equal(run_native_port_threaded(A, B, C, threads=4), run_native_port(A, B, C))


def test_fp64_run_native_equals_naive():
    """The reference's native body is bitwise naive_gemm in fp64 (same order, same rounding)."""
    cases = [c for c in golden_cases() if c["precision"] == "double"]
    assert cases and all(c["run_native_bitwise_naive"] for c in cases)


def test_known_answers():
    assert naive_gemm(np.array([[2.0]]), np.array([[3.0]]), np.array([[5.0]]))[0, 0] == 11.0
    got = naive_gemm(np.array([[1.0, 1.0]], np.float32), np.array([[2.0 ** 14], [2.0 ** -11]], np.float32),
                     np.zeros((1, 1), np.float32))[0, 0]
    assert got == np.float32(np.float64(2.0 ** 14) + np.float64(2.0 ** -11))
    with pytest.raises(ValueError):
        naive_gemm(np.ones((4, 4)), np.ones((4, 2)), np.ones((4, 3)))


def test_row_slab_is_exact_restriction():
    rng = np.random.default_rng(2)
    A, B, C = rng.random((500, 200)), rng.random((200, 4)), rng.random((500, 4))
    full = naive_gemm(A, B, C)
    assert np.array_equal(naive_gemm(A[100:200], B, C[100:200]), full[100:200])
