"""GPU parity: the sm_100a kernels against the CPU oracle (oracle/reference.py, itself pinned to
the reference package by tests/test_oracle_golden.py).

Tolerances (BASELINE.json north_star): relative Frobenius error <= 1e-12 (fp64), <= 1e-5 (fp32);
plus the reference's own acceptance bound max_rel_error <= 8*k*eps (test_acceptance.py:72-74).
Exact cases (identity, zero B, small integers) must be bitwise.
"""

import zlib

import numpy as np
import pytest

from conftest import TOL_FROB, golden_cases, regenerate
from oracle import max_rel_error, naive_gemm, rel_frobenius

pytestmark = pytest.mark.gpu

EXACT = {"identity_v3", "zero_b_v0", "scalar_fma", "single_accumulates_double"}


def _tsm():
    import paper_2002_03258_b200 as tsm
    return tsm


def _mat(tsm, X, prec):
    return tsm.Matrix(X.shape[0], X.shape[1], X.reshape(-1, order="F"), prec)


def _check(out2d, ref2d, k, precision, exact=False, what=""):
    if exact:
        assert np.array_equal(out2d, ref2d), what
        return
    eps = np.finfo(np.float64 if precision == "double" else np.float32).eps
    fro = rel_frobenius(out2d, ref2d)
    mre = max_rel_error(out2d, ref2d)
    assert fro <= TOL_FROB[precision], (what, fro)
    assert mre <= 8 * k * eps, (what, mre)


@pytest.mark.parametrize("case", golden_cases(), ids=lambda c: c["name"])
def test_run_native_golden(case):
    """Every golden case through the drop-in run_native (host Matrix in/out)."""
    tsm = _tsm()
    A, B, C0 = regenerate(case)
    prec = tsm.Precision.parse(case["precision"])
    p = case["params"]
    variant = tsm.Variant.parse(case["variant"])
    params = tsm.KernelParams(t1=p["t1"], t2=p["t2"], t3=p["t3"], tcf=p["tcf"], variant=variant)
    out = tsm.run_native(variant, _mat(tsm, A, prec), _mat(tsm, B, prec), _mat(tsm, C0, prec), params)
    assert isinstance(out, tsm.Matrix) and out.rows == case["m"] and out.cols == case["n"]
    assert not out.storage.flags.writeable
    ref = naive_gemm(A, B, C0)
    _check(out.to_2d(), ref, case["k"], case["precision"], exact=case["name"] in EXACT, what=case["name"])


@pytest.mark.parametrize("impl", ["auto", "ldg", "tma", "tsm2l", "ablation"])
@pytest.mark.parametrize("variant", ["v0", "v1", "v2", "v3", "l-opt1", "l-opt2"])
def test_device_impls_ragged(impl, variant):
    """Device API, every implementation x variant, ragged shapes, odd leading dimensions."""
    import torch
    tsm = _tsm()
    rng = np.random.default_rng(zlib.crc32(f"{impl}/{variant}".encode()))
    for (m, k, n) in [(1, 1, 1), (37, 5, 3), (333, 61, 7), (1025, 257, 16), (700, 1999, 9), (4099, 64, 2)]:
        if impl == "tsm2l" and k > 64:
            continue
        for dtype in (np.float64, np.float32):
            A = rng.random((m, k)).astype(dtype)
            B = rng.random((k, n)).astype(dtype)
            C0 = np.zeros((m, n), dtype) if variant == "l-opt2" else rng.random((m, n)).astype(dtype)
            dev = torch.device("cuda")
            # odd leading dimension on purpose: exercises the scalar / LDG paths
            lda = m + (1 if m % 2 else 3)
            At = torch.zeros((k, lda), dtype=torch.from_numpy(A).dtype, device=dev).t()[:m]
            At.copy_(torch.from_numpy(A))
            Bt = torch.from_numpy(np.asfortranarray(B)).to(dev).t().contiguous().t()
            Ct = torch.from_numpy(np.asfortranarray(C0)).to(dev).t().contiguous().t()
            tsm.gemm(At, Bt, Ct, variant=variant, impl=impl, c_is_zero=(variant == "l-opt2"),
                     params=tsm.KernelParams(t1=64, t2=1, t3=4, tcf=1, variant=tsm.Variant.parse(variant)))
            torch.cuda.synchronize()
            prec = "double" if dtype == np.float64 else "single"
            _check(Ct.cpu().numpy(), naive_gemm(A, B, C0), k, prec, what=(impl, variant, m, k, n, prec))


@pytest.mark.parametrize("det", [False, True])
def test_aligned_tma_many_shapes(det):
    """The TMA path on padded (aligned) layouts, covering k tails, row tails and split row blocks,
    for the dynamic (default) and the deterministic static-split kernels."""
    import torch
    tsm = _tsm()
    rng = np.random.default_rng(7)
    shapes = [(512, 8, 4), (513, 9, 4), (4096, 4096, 8), (1000, 3001, 16), (64, 20000, 2), (5000, 100, 1),
              (2049, 777, 12), (30, 65, 16)]
    for (m, k, n) in shapes:
        for dt in (torch.float64, torch.float32):
            A = tsm.colmajor_empty(m, k, dt, "cuda")
            A.copy_(torch.from_numpy(rng.random((m, k))).to(dt))
            B = tsm.colmajor_empty(k, n, dt, "cuda")
            B.copy_(torch.from_numpy(rng.random((k, n))).to(dt))
            C = tsm.colmajor_empty(m, n, dt, "cuda")
            C0 = rng.random((m, n))
            C.copy_(torch.from_numpy(C0).to(dt))
            tsm.gemm(A, B, C, impl="tma", deterministic=det)
            torch.cuda.synchronize()
            An, Bn = A.cpu().numpy(), B.cpu().numpy()
            ref = naive_gemm(An, Bn, C0.astype(An.dtype))
            _check(C.cpu().numpy(), ref, k, "double" if dt == torch.float64 else "single", what=(m, k, n, dt))


def test_dynamic_queue_item_counts():
    """Split shapes whose item count is at / below / just above the CTA count (some CTAs get no
    item at all — the end-of-work marker must still release them), and tiny single-item ones."""
    import torch
    tsm = _tsm()
    rng = np.random.default_rng(17)
    for (m, k, n) in [(1024, 1024, 16), (1024, 1024, 8), (512, 300, 8), (1500, 2000, 16), (300, 5000, 4),
                      (10000, 700, 16), (513, 4000, 9), (64, 129, 1)]:
        for dt in (torch.float64, torch.float32):
            A = tsm.colmajor_empty(m, k, dt, "cuda")
            A.copy_(torch.from_numpy(rng.random((m, k))).to(dt))
            B = tsm.colmajor_empty(k, n, dt, "cuda")
            B.copy_(torch.from_numpy(rng.random((k, n))).to(dt))
            C = tsm.colmajor_empty(m, n, dt, "cuda")
            C0 = rng.random((m, n))
            C.copy_(torch.from_numpy(C0).to(dt))
            for _ in range(3):  # repeated launches reuse the queue / workspace
                tsm.gemm(A, B, C)
            torch.cuda.synchronize()
            An, Bn = A.cpu().numpy(), B.cpu().numpy()
            ref = C0.astype(An.dtype)
            for _ in range(3):
                ref = naive_gemm(An, Bn, ref)
            _check(C.cpu().numpy(), ref, 3 * k, "double" if dt == torch.float64 else "single", what=(m, k, n, dt))


@pytest.mark.parametrize("dt", ["float64", "float32"])
def test_deterministic_repeat(dt):
    """deterministic=True (static split, fixed-order combine): launches give bitwise-identical C;
    the default dynamic kernel agrees with it within tolerance."""
    import torch
    tsm = _tsm()
    m, k, n = 6000, 20000, 8
    dtype = getattr(torch, dt)
    A = tsm.colmajor_empty(m, k, dtype, "cuda")
    tsm.fill_uniform(A, seed=11)
    B = tsm.colmajor_empty(k, n, dtype, "cuda")
    tsm.fill_uniform(B, seed=12)
    from paper_2002_03258_b200 import tuning
    outs = []
    for det in (True, True, True, False):
        C = tsm.colmajor_empty(m, n, dtype, "cuda")
        C.fill_(1.0)
        tsm.gemm(A, B, C, deterministic=det)
        outs.append(C.cpu().numpy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    _check(outs[3], outs[0].astype(np.float64), k, "double" if dt == "float64" else "single")
    # the static stream-K split (combine=3) is reproducible too; chunk-ordered (combine=1) is
    # what deterministic=True selects
    try:
        for combine in (3, 1):
            tuning.set_tuning(tuning.Tuning(combine=combine))
            rep = []
            for _ in range(2):
                C = tsm.colmajor_empty(m, n, dtype, "cuda")
                C.fill_(1.0)
                tsm.gemm(A, B, C)
                rep.append(C.cpu().numpy())
            assert np.array_equal(rep[0], rep[1]), combine
            _check(rep[0], outs[0].astype(np.float64), k, "double" if dt == "float64" else "single")
        assert np.array_equal(rep[0], outs[0])  # combine=1 is what deterministic=True runs
    finally:
        tuning.set_tuning(None)


def test_fill_uniform_matches_host_rng():
    import torch
    from oracle.rng import uniform_block
    tsm = _tsm()
    for dt, npdt in ((torch.float64, np.float64), (torch.float32, np.float32)):
        T = tsm.colmajor_empty(300, 7, dt, "cuda")
        tsm.fill_uniform(T, seed=2024, row_offset=1000, col_offset=5)
        host = uniform_block(range(1000, 1300), range(5, 12), 2024, npdt)
        assert np.array_equal(T.cpu().numpy(), host)


def test_l_opt2_nonzero_c_rejected():
    tsm = _tsm()
    A = tsm.Matrix.from_2d(np.ones((256, 8)), tsm.Precision.DOUBLE)
    B = tsm.Matrix.from_2d(np.ones((8, 8)), tsm.Precision.DOUBLE)
    C = tsm.Matrix.from_2d(np.ones((256, 8)), tsm.Precision.DOUBLE)
    p = tsm.KernelParams(t1=32, t2=8, t3=4, tcf=2, variant=tsm.Variant.L_OPT2)
    with pytest.raises(ValueError):
        tsm.run_native(tsm.Variant.L_OPT2, A, B, C, p)


def test_l_opt2_device_check():
    import torch
    tsm = _tsm()
    A = torch.ones((64, 4), dtype=torch.float64, device="cuda").t().contiguous().t()
    B = torch.ones((4, 4), dtype=torch.float64, device="cuda").t()
    C = torch.ones((64, 4), dtype=torch.float64, device="cuda").t().contiguous().t()
    with pytest.raises(ValueError):
        tsm.gemm(A, B, C, variant="l-opt2", check_zero_c=True)
    C.zero_()
    tsm.gemm(A, B, C, variant="l-opt2", check_zero_c=True)
    assert torch.all(C == 4.0)


@pytest.mark.parametrize("variant", ["v3", "l-opt1", "l-opt2"])
@pytest.mark.parametrize("prec", ["double", "single"])
def test_run_native_host_path_shapes(variant, prec):
    """run_native (host Matrix in/out) across TSM2R/TSM2L shapes, both precisions, n > 16,
    nonzero C (except L_OPT2), including fp32 split row blocks (fp64 accumulator + finalize)."""
    tsm = _tsm()
    rng = np.random.default_rng(zlib.crc32(f"{variant}/{prec}".encode()))
    dt = np.float64 if prec == "double" else np.float32
    for (m, k, n) in [(5000, 6000, 8), (3001, 9000, 17), (100000, 16, 16), (40000, 40, 3)]:
        A = rng.random((m, k)).astype(dt)
        B = rng.random((k, n)).astype(dt)
        C0 = np.zeros((m, n), dt) if variant == "l-opt2" else rng.random((m, n)).astype(dt)
        v = tsm.Variant.parse(variant)
        p = tsm.KernelParams(t1=128, t2=min(4, n), t3=4, tcf=2 if v.is_tsm2l else 1, variant=v)
        out = tsm.run_native(v, tsm.Matrix.from_2d(A, prec), tsm.Matrix.from_2d(B, prec),
                             tsm.Matrix.from_2d(C0, prec), p)
        _check(out.to_2d(), naive_gemm(A, B, C0), k, prec, what=(variant, prec, m, k, n))


def test_accepts_reference_objects_duck_typed():
    """run_native takes objects shaped like the reference's Matrix/KernelParams (rows, cols,
    storage, precision.value; t1..tcf, variant.value)."""
    import types
    tsm = _tsm()
    rng = np.random.default_rng(9)
    A, B = rng.random((300, 200)), rng.random((200, 4))
    prec = types.SimpleNamespace(value="double")

    def mat(X):
        return types.SimpleNamespace(rows=X.shape[0], cols=X.shape[1], storage=X.reshape(-1, order="F"),
                                     precision=prec)
    params = types.SimpleNamespace(t1=128, t2=4, t3=4, tcf=1, variant=types.SimpleNamespace(value="v3"))
    out = tsm.run_native(types.SimpleNamespace(value="v3"), mat(A), mat(B), mat(np.zeros((300, 4))), params)
    _check(out.to_2d(), naive_gemm(A, B, np.zeros((300, 4))), 200, "double")


def test_wide_n_multi_pass():
    """n > 16 runs as 16-wide passes (A re-read per pass, as the paper's t2 passes)."""
    tsm = _tsm()
    rng = np.random.default_rng(3)
    for (m, k, n) in [(700, 300, 40), (3000, 40, 33), (5000, 2000, 20)]:
        for prec, dt in (("double", np.float64), ("single", np.float32)):
            # fp32: 16-column passes on the tensor cores, the remainder pass on FFMA2
            A, B, C0 = (rng.random((m, k)).astype(dt), rng.random((k, n)).astype(dt), rng.random((m, n)).astype(dt))
            out = tsm.run_native(tsm.Variant.V3, tsm.Matrix.from_2d(A, prec), tsm.Matrix.from_2d(B, prec),
                                 tsm.Matrix.from_2d(C0, prec), tsm.KernelParams(t2=4))
            _check(out.to_2d(), naive_gemm(A, B, C0), k, prec, what=(m, k, n, prec))


def test_host_path_pinned_and_pageable_slabs():
    """run_host with several H2D slabs (TSM2R column slabs, TSM2L row slabs), pinned and pageable."""
    import ctypes
    import torch
    from paper_2002_03258_b200 import _lib
    rng = np.random.default_rng(4)
    for (m, k, n) in [(8192, 9000, 8), (3_000_000, 16, 16)]:
        A = np.asfortranarray(rng.random((m, k)))
        B = np.asfortranarray(rng.random((k, n)))
        C0 = np.asfortranarray(rng.random((m, n)))
        for pinned in (False, True):
            if pinned:
                At = torch.from_numpy(A.T.copy()).pin_memory()  # (k, m) row-major == A column-major
                a_ptr = At.data_ptr()
            else:
                a_ptr = A.ctypes.data
            out = np.empty((m, n), order="F")
            p = _lib.Params(128, 4, 4, 1, 3)
            rc = _lib.load().tsm2x_run_host(3, _lib.DOUBLE, m, k, n, a_ptr, m, B.ctypes.data, k, C0.ctypes.data,
                                            out.ctypes.data, m, ctypes.byref(p), 0, 0)
            _lib.check(rc)
            rows = np.r_[0:64, m // 2:m // 2 + 64, m - 64:m]
            ref = naive_gemm(A[rows], B, C0[rows])
            _check(out[rows], ref, k, "double", what=(m, k, n, pinned))


@pytest.mark.parametrize("m,k,n,prec", [(6144, 6144, 16, "double"), (16384, 16384, 8, "double"),
                                         (12345, 9999, 13, "double"), (8192, 8192, 16, "single"),
                                         (700, 3000, 16, "single"), (1000, 200, 8, "double")])
def test_equal_split_regimes(m, k, n, prec):
    """The equal-item split (make_items: up to 24 MB of A per CTA, or fewer row blocks than SMs):
    one round, several rounds (16384^2: 288 items on 148 CTAs), ragged rows / columns, and the
    short-k shapes that used to stay on one CTA — sampled row slabs against the oracle and the
    whole result against cuBLAS, with C += A·B over a nonzero C."""
    import torch
    from oracle.rng import uniform_block
    tsm = _tsm()
    dt = torch.float64 if prec == "double" else torch.float32
    npdt = np.float64 if prec == "double" else np.float32
    A = tsm.colmajor_empty(m, k, dt, "cuda")
    tsm.fill_uniform(A, seed=31)
    B = tsm.colmajor_empty(k, n, dt, "cuda")
    tsm.fill_uniform(B, seed=32)
    C = tsm.colmajor_empty(m, n, dt, "cuda")
    tsm.fill_uniform(C, seed=33)
    C0 = C.clone()
    tsm.gemm(A, B, C)
    torch.cuda.synchronize()
    Bh = uniform_block(range(k), range(n), 32).astype(npdt)
    Ch = C.cpu().numpy()
    C0h = C0.cpu().numpy()
    for r0 in sorted({0, m // 3, max(0, m - 97)}):
        rows = range(r0, min(m, r0 + 97))
        Ah = uniform_block(rows, range(k), 31).astype(npdt)
        ref = naive_gemm(Ah, Bh, C0h[r0:r0 + len(rows)])
        _check(Ch[r0:r0 + len(rows)], ref, k, prec, what=("slab", m, k, n, r0))
    full = (C0.double() + A.double() @ B.double()).cpu().numpy()
    assert rel_frobenius(Ch, full) <= (1e-12 if prec == "double" else 1e-5)


@pytest.mark.slow
@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_config2_sampled_rows(n):
    """BASELINE config 2 (ref m=k=30720, n=2..16, fp64) at full size: sampled row slabs against
    the oracle (rows are independent, so slabs are exact restrictions) and the full result
    against cuBLAS DGEMM (relative Frobenius)."""
    import torch
    from oracle.rng import uniform_block
    tsm = _tsm()
    m = k = 30720
    A = tsm.colmajor_empty(m, k, torch.float64, "cuda")
    tsm.fill_uniform(A, seed=2024)
    B = tsm.colmajor_empty(k, n, torch.float64, "cuda")
    tsm.fill_uniform(B, seed=2025)
    C = tsm.colmajor_empty(m, n, torch.float64, "cuda")
    C.zero_()
    tsm.gemm(A, B, C, c_is_zero=True)
    torch.cuda.synchronize()
    Bh = uniform_block(range(k), range(n), 2025)
    Ch = C.cpu().numpy()
    for r0 in (0, 12345, m - 256):
        rows = range(r0, r0 + 256)
        Ah = uniform_block(rows, range(k), 2024)
        ref = naive_gemm(Ah, Bh, np.zeros((256, n)))
        _check(Ch[r0:r0 + 256], ref, k, "double", what=("slab", r0))
    full = (A @ B).cpu().numpy()
    assert rel_frobenius(Ch, full) <= 1e-12


@pytest.mark.slow
def test_config5_per_gpu_shard_sampled():
    """BASELINE config 5 per GPU (ref m=k=65536, n=8, fp64; 34 GB of A) — the largest single-GPU
    problem — sampled row slabs against the oracle, plus a rank-1 shard of the 2-GPU split
    generated with its global row offset (what each rank of the multi-GPU run computes)."""
    import torch
    from oracle.rng import uniform_block
    tsm = _tsm()
    m = k = 65536
    n = 8
    A = tsm.colmajor_empty(m, k, torch.float64, "cuda")
    tsm.fill_uniform(A, seed=5)
    B = tsm.colmajor_empty(k, n, torch.float64, "cuda")
    tsm.fill_uniform(B, seed=6)
    C = tsm.colmajor_empty(m, n, torch.float64, "cuda")
    C.zero_()
    tsm.gemm(A, B, C, c_is_zero=True)
    torch.cuda.synchronize()
    Ch = C.cpu().numpy()
    del A
    torch.cuda.empty_cache()
    Bh = uniform_block(range(k), range(n), 6)
    for r0 in (0, 40000, m - 128):
        rows = range(r0, r0 + 128)
        ref = naive_gemm(uniform_block(rows, range(k), 5), Bh, np.zeros((128, n)))
        _check(Ch[r0:r0 + 128], ref, k, "double", what=("config5", r0))
    # the second half as its own shard (global row offset) agrees with the full run's rows
    from paper_2002_03258_b200.multi import row_partition
    s0, s1 = row_partition(m, 2, 1)
    As = tsm.colmajor_empty(s1 - s0, k, torch.float64, "cuda")
    tsm.fill_uniform(As, seed=5, row_offset=s0)
    Cs = tsm.colmajor_empty(s1 - s0, n, torch.float64, "cuda")
    Cs.zero_()
    tsm.gemm(As, B, Cs, c_is_zero=True, deterministic=True)
    torch.cuda.synchronize()
    _check(Cs.cpu().numpy(), Ch[s0:s1], k, "double", what="shard")


@pytest.mark.slow
def test_config3_tsm2l_sampled():
    import torch
    from oracle.rng import uniform_block
    tsm = _tsm()
    m, k, n = 1 << 24, 16, 16
    A = tsm.colmajor_empty(m, k, torch.float64, "cuda")
    tsm.fill_uniform(A, seed=7)
    B = tsm.colmajor_empty(k, n, torch.float64, "cuda")
    tsm.fill_uniform(B, seed=8)
    C = tsm.colmajor_empty(m, n, torch.float64, "cuda")
    tsm.fill_uniform(C, seed=9)
    tsm.gemm(A, B, C, variant="l-opt1")
    torch.cuda.synchronize()
    Bh = uniform_block(range(k), range(n), 8)
    for r0 in (0, m // 3, m - 1000):
        rows = range(r0, r0 + 1000)
        ref = naive_gemm(uniform_block(rows, range(k), 7), Bh, uniform_block(rows, range(n), 9))
        _check(C[r0:r0 + 1000].cpu().numpy(), ref, k, "double", what=r0)


@pytest.mark.slow
def test_config4_fp32_sampled():
    import torch
    from oracle.rng import uniform_block
    tsm = _tsm()
    m = k = 32768
    n = 16
    A = tsm.colmajor_empty(m, k, torch.float32, "cuda")
    tsm.fill_uniform(A, seed=31)
    B = tsm.colmajor_empty(k, n, torch.float32, "cuda")
    tsm.fill_uniform(B, seed=32)
    C = tsm.colmajor_empty(m, n, torch.float32, "cuda")
    C.zero_()
    tsm.gemm(A, B, C, c_is_zero=True)
    torch.cuda.synchronize()
    Ch = C.cpu().numpy()
    Bh = uniform_block(range(k), range(n), 32, np.float32)
    for r0 in (0, m - 128):
        rows = range(r0, r0 + 128)
        ref = naive_gemm(uniform_block(rows, range(k), 31, np.float32), Bh, np.zeros((128, n), np.float32))
        _check(Ch[r0:r0 + 128], ref, k, "single", what=r0)


@pytest.mark.slow
def test_config4_fp32_benchmarked_path_full():
    """BASELINE config 4 exactly as benchmarked (fp32 32768^2 x 16, C += A*B with a nonzero C; the
    split-precision tf32 tcgen05 path with fp64 split-row-block combine): the FULL result against
    an fp64 cuBLAS product of the same device inputs (relative Frobenius <= 1e-5, and the max
    relative error bound), plus 8 row slabs spread over the split row blocks against the oracle."""
    import torch
    from oracle.rng import uniform_block
    tsm = _tsm()
    m = k = 32768
    n = 16
    A = tsm.colmajor_empty(m, k, torch.float32, "cuda")
    tsm.fill_uniform(A, seed=41)
    B = tsm.colmajor_empty(k, n, torch.float32, "cuda")
    tsm.fill_uniform(B, seed=42)
    C = tsm.colmajor_empty(m, n, torch.float32, "cuda")
    tsm.fill_uniform(C, seed=43)
    C0 = C.clone()
    from paper_2002_03258_b200 import tuning
    plan = tuning.plan("single", m, k, n)
    assert plan["consumer"] == "tc" and plan["nbig"] + plan["nsmall"] > 1  # split row blocks, tcgen05
    tsm.gemm(A, B, C)
    torch.cuda.synchronize()
    Ch = C.cpu().numpy()
    full = (C0.double() + A.double() @ B.double()).cpu().numpy()
    assert rel_frobenius(Ch, full) <= 1e-5
    assert max_rel_error(Ch, full) <= 8 * k * np.finfo(np.float32).eps
    assert np.isfinite(Ch).all()
    del A
    torch.cuda.empty_cache()
    Bh = uniform_block(range(k), range(n), 42, np.float32)
    C0h = C0.cpu().numpy()
    for r0 in np.linspace(0, m - 64, 8).astype(int):
        rows = range(int(r0), int(r0) + 64)
        ref = naive_gemm(uniform_block(rows, range(k), 41, np.float32), Bh, C0h[r0:r0 + 64])
        _check(Ch[r0:r0 + 64], ref, k, "single", what=("config4 slab", int(r0)))


@pytest.mark.slow
@pytest.mark.parametrize("prec", ["double", "single"])
def test_config3_l_opt2_zero_c_benchmarked_path(prec):
    """BASELINE config 3 as benchmarked: L_OPT2 (zero-C contract, C never read) at m = 2^24,
    k = n = 16 — fp64 (DMMA) and fp32 (FFMA2 single-chunk path with the direct-store epilogue):
    full result against a float64 torch product of the same inputs and sampled slabs against the
    oracle. C starts as NaN so a read of C would show."""
    import torch
    from oracle.rng import uniform_block
    tsm = _tsm()
    dt = torch.float64 if prec == "double" else torch.float32
    tol = 1e-12 if prec == "double" else 1e-5
    m, k, n = 1 << 24, 16, 16
    A = tsm.colmajor_empty(m, k, dt, "cuda")
    tsm.fill_uniform(A, seed=17)
    B = tsm.colmajor_empty(k, n, dt, "cuda")
    tsm.fill_uniform(B, seed=18)
    C = tsm.colmajor_empty(m, n, dt, "cuda")
    C.fill_(float("nan"))  # c_is_zero: the kernel must not read it
    tsm.gemm(A, B, C, variant="l-opt2", c_is_zero=True)
    torch.cuda.synchronize()
    full = A.double() @ B.double()
    assert torch.isfinite(C).all()
    assert rel_frobenius(C.double().cpu().numpy(), full.cpu().numpy()) <= tol
    npdt = np.float64 if prec == "double" else np.float32
    Bh = uniform_block(range(k), range(n), 18).astype(npdt)
    for r0 in (0, 5_000_017, m - 777):
        rows = range(r0, min(m, r0 + 777))
        ref = naive_gemm(uniform_block(rows, range(k), 17).astype(npdt), Bh, np.zeros((len(rows), n), npdt))
        _check(C[r0:r0 + len(rows)].cpu().numpy(), ref, k, prec, what=("l-opt2", prec, r0))


@pytest.mark.parametrize("consumer", ["fma", "dmma", "ffma2", "tc", "dmmap", "dmma/cw16", "fma/cw16", "auto/sb64",
                                      "dmma/sb64", "auto/inline0", "auto/inline1", "fma/inline1", "dmmap/inline1",
                                      "ffma2/inline1", "dmma/sb64/inline1"])
def test_consumer_policies_subprocess(consumer):
    """Each TMA consumer policy (TSM2X_CONSUMER override; "/cw16" = the 16-consumer-warp x 1-row
    geometry, TSM2X_CW=16 TSM2X_RPT=1) on split and single-chunk shapes; "/inline0" / "/inline1"
    force the prep-kernel / inline-B producer (TSM2X_INLINE_B) for every call."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_2002_03258_b200 as tsm
from oracle import naive_gemm, rel_frobenius
rng = np.random.default_rng(5)
for (m, k, n) in [(2000, 5000, 16), (1500, 3001, 8), (777, 10000, 12), (4096, 16, 16), (513, 20000, 3),
                  (70001, 16, 16), (5000, 24, 8)]:
    for dt in (torch.float64, torch.float32):
        A = tsm.colmajor_empty(m, k, dt, "cuda"); A.copy_(torch.from_numpy(rng.random((m, k))).to(dt))
        B = tsm.colmajor_empty(k, n, dt, "cuda"); B.copy_(torch.from_numpy(rng.random((k, n))).to(dt))
        C = tsm.colmajor_empty(m, n, dt, "cuda"); C0 = rng.random((m, n)); C.copy_(torch.from_numpy(C0).to(dt))
        czero = k <= 24 and n % 2 == 0  # single-chunk shapes: also the zero-C contract (C never read)
        if czero:
            C.zero_(); C0 = np.zeros((m, n))
        tsm.gemm(A, B, C, variant="l-opt2" if czero else "v3", c_is_zero=czero)
        ref = naive_gemm(A.cpu().numpy(), B.cpu().numpy(), C0.astype(A.cpu().numpy().dtype))
        err = rel_frobenius(C.cpu().numpy(), ref)
        tol = 1e-12 if dt == torch.float64 else 1e-5
        assert err <= tol, (m, k, n, dt, err)
print("ok")
'''
    env = dict(os.environ)
    if not consumer.startswith("auto"):
        env["TSM2X_CONSUMER"] = consumer.split("/")[0]
    if consumer.endswith("/cw16"):
        env.update(TSM2X_CW="16", TSM2X_RPT="1")
    if "/sb64" in consumer:  # 64 KB pipeline stages (fp64 8/16-column passes)
        env.update(TSM2X_STAGE_KB="64")
    if "/inline" in consumer:
        env["TSM2X_INLINE_B"] = consumer.split("/inline")[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stdout + out.stderr


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_run_native_multi_device_shards(devices):
    """tsm2x_run_host_multi: row shards on (repeated) devices, TSM2R and TSM2L, nonzero C."""
    tsm = _tsm()
    rng = np.random.default_rng(len(devices))
    for (m, k, n) in [(4099, 3000, 8), (70001, 16, 16), (33, 100, 3)]:
        A, B, C0 = rng.random((m, k)), rng.random((k, n)), rng.random((m, n))
        out = tsm.run_native_multi(tsm.Variant.V3, tsm.Matrix.from_2d(A, "double"), tsm.Matrix.from_2d(B, "double"),
                                   tsm.Matrix.from_2d(C0, "double"), tsm.KernelParams(t2=min(4, n)), devices)
        _check(out.to_2d(), naive_gemm(A, B, C0), k, "double", what=(devices, m, k, n))


@pytest.mark.parametrize("c_zero", [False, True])
def test_tc32_tensor_core_shapes(c_zero):
    """fp32 16-column passes on the tensor cores (tsm2r_stream_tc32, split-precision tf32): ragged
    rows (m % 32, m % 512), ragged k (k % 16), n = 9..16, split and single-chunk row blocks,
    C += A.B and the zero-C contract. Auto sends single-chunk row blocks to FFMA2, so the tensor
    cores are forced (tuning consumer 4) to cover their single-chunk instantiation too."""
    import torch
    tsm = _tsm()
    from paper_2002_03258_b200 import tuning
    rng = np.random.default_rng(11 + c_zero)
    tuning.set_tuning(tuning.Tuning(consumer=4))
    try:
        _tc32_shapes(tsm, tuning, rng, c_zero, torch)
    finally:
        tuning.set_tuning(None)


def _tc32_shapes(tsm, tuning, rng, c_zero, torch):
    for (m, k, n) in [(1, 1, 16), (31, 7, 9), (33, 17, 12), (513, 100, 16), (4113, 5000, 16), (1024, 33, 15),
                      (70001, 16, 16), (2048, 40000, 16)]:
        assert tuning.plan("single", m, k, n)["consumer"] == "tc", (m, k, n)
        A = tsm.colmajor_empty(m, k, torch.float32, "cuda")
        A.copy_(torch.from_numpy(rng.standard_normal((m, k)).astype(np.float32)))
        B = tsm.colmajor_empty(k, n, torch.float32, "cuda")
        B.copy_(torch.from_numpy(rng.standard_normal((k, n)).astype(np.float32)))
        C0 = np.zeros((m, n), np.float32) if c_zero else rng.standard_normal((m, n)).astype(np.float32)
        C = tsm.colmajor_empty(m, n, torch.float32, "cuda")
        C.copy_(torch.from_numpy(C0))
        tsm.gemm(A, B, C, variant="l-opt2" if c_zero else "v3", c_is_zero=c_zero)
        ref = naive_gemm(A.cpu().numpy().astype(np.float64), B.cpu().numpy().astype(np.float64), C0.astype(np.float64))
        out = C.cpu().numpy().astype(np.float64)
        assert rel_frobenius(out, ref) <= 1e-5, (m, k, n, rel_frobenius(out, ref))
        # elementwise: within fp32 accumulation error of the |A||B| scale
        scale = np.abs(A.cpu().numpy()).astype(np.float64) @ np.abs(B.cpu().numpy()).astype(np.float64) + np.abs(C0)
        assert np.max(np.abs(out - ref) / scale) <= 4 * k * np.finfo(np.float32).eps + 1e-6, (m, k, n)


def test_tc32_exact_cases():
    """Tensor-core fp32 path: small integers are exact; an identity A returns B to within the
    split's one dropped term (lo(B) enters as tf32: 2^-22 relative) — the bitwise identity of the
    reference's tests (test_kernels.py:20-44) is fp64, which stays bitwise (golden identity_v3)."""
    import torch
    tsm = _tsm()
    rng = np.random.default_rng(3)
    k, n = 256, 16
    Bh = rng.standard_normal((k, n)).astype(np.float32)
    A = tsm.colmajor_empty(k, k, torch.float32, "cuda")
    A.copy_(torch.eye(k))
    B = tsm.colmajor_empty(k, n, torch.float32, "cuda")
    B.copy_(torch.from_numpy(Bh))
    C = tsm.colmajor_empty(k, n, torch.float32, "cuda")
    C.zero_()
    tsm.gemm(A, B, C)
    assert np.max(np.abs(C.cpu().numpy() - Bh) / np.abs(Bh)) <= 2.0 ** -21
    Ai = rng.integers(-8, 8, (1000, 640)).astype(np.float32)
    Bi = rng.integers(-8, 8, (640, 16)).astype(np.float32)
    A = tsm.colmajor_empty(1000, 640, torch.float32, "cuda")
    A.copy_(torch.from_numpy(Ai))
    B = tsm.colmajor_empty(640, 16, torch.float32, "cuda")
    B.copy_(torch.from_numpy(Bi))
    C = tsm.colmajor_empty(1000, 16, torch.float32, "cuda")
    C.zero_()
    tsm.gemm(A, B, C)
    assert np.array_equal(C.cpu().numpy(), Ai @ Bi)


def test_tc32_nonfinite_inputs_propagate():
    """Non-finite entries of A or B give non-finite outputs in exactly the reference's positions
    (an infinity may surface as NaN on the tensor-core path: inf * 0 in the split cross terms);
    deterministic=True (FFMA2, IEEE fp32 FMA chain) matches the reference's inf/NaN kinds too."""
    import torch
    tsm = _tsm()
    rng = np.random.default_rng(5)
    m, k, n = 600, 300, 16
    Ah = rng.random((m, k)).astype(np.float32)
    Bh = rng.random((k, n)).astype(np.float32)
    Ah[5, 7] = np.inf
    Ah[100, 0] = -np.inf
    Ah[300, 299] = np.nan
    Bh[11, 3] = np.inf
    with np.errstate(invalid="ignore", over="ignore"):
        ref = Ah.astype(np.float64) @ Bh.astype(np.float64)
    for det in (False, True):
        A = tsm.colmajor_empty(m, k, torch.float32, "cuda")
        A.copy_(torch.from_numpy(Ah))
        B = tsm.colmajor_empty(k, n, torch.float32, "cuda")
        B.copy_(torch.from_numpy(Bh))
        C = tsm.colmajor_empty(m, n, torch.float32, "cuda")
        C.zero_()
        tsm.gemm(A, B, C, deterministic=det)
        out = C.cpu().numpy()
        assert np.array_equal(~np.isfinite(out), ~np.isfinite(ref)), det
        fin = np.isfinite(ref)
        assert rel_frobenius(out[fin].astype(np.float64), ref[fin]) <= 1e-5
        if det:
            assert np.array_equal(np.isnan(out), np.isnan(ref))


def test_tsm2l_zero_c_shapes():
    """TSM2L under the zero-C contract (L_OPT2), fp64 8/16-column passes (DMMA consumer,
    single-chunk row blocks, 16-byte row-pair stores): ragged rows, k = 9..64, w = 9..16."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_2002_03258_b200 as tsm
from oracle import naive_gemm, rel_frobenius
rng = np.random.default_rng(9)
for (m, k, n) in [(1, 16, 16), (700, 16, 16), (70001, 16, 16), (5000, 9, 12), (4096, 64, 16), (513, 17, 9),
                  (100000, 24, 16)]:
    A = tsm.colmajor_empty(m, k, torch.float64, "cuda"); A.copy_(torch.from_numpy(rng.standard_normal((m, k))))
    B = tsm.colmajor_empty(k, n, torch.float64, "cuda"); B.copy_(torch.from_numpy(rng.standard_normal((k, n))))
    C = tsm.colmajor_empty(m, n, torch.float64, "cuda"); C.fill_(7.0)
    C.zero_()
    tsm.gemm(A, B, C, variant="l-opt2", c_is_zero=True)
    ref = naive_gemm(A.cpu().numpy(), B.cpu().numpy(), np.zeros((m, n)))
    err = rel_frobenius(C.cpu().numpy(), ref)
    assert err <= 1e-12, (m, k, n, err)
print("ok")
'''
    env = dict(os.environ)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stdout + out.stderr


def test_cuda_graph_capture_and_replay():
    """The device API is stream-ordered and capture-safe: tsm.gemm captured into a CUDA graph
    (workspace from the stream-ordered allocator, work queue reset by the kernel itself) replays
    to the same result, for TSM2R fp64 (split row blocks, fp64 reductions), fp32 on the tensor
    cores, and TSM2L."""
    import torch
    tsm = _tsm()
    rng = np.random.default_rng(21)
    for (m, k, n, dt, variant) in [(4096, 4096, 8, torch.float64, "v3"), (4096, 3000, 16, torch.float32, "v3"),
                                   (70000, 16, 16, torch.float64, "l-opt2")]:
        A = tsm.colmajor_empty(m, k, dt, "cuda")
        A.copy_(torch.from_numpy(rng.random((m, k))).to(dt))
        B = tsm.colmajor_empty(k, n, dt, "cuda")
        B.copy_(torch.from_numpy(rng.random((k, n))).to(dt))
        C = tsm.colmajor_empty(m, n, dt, "cuda")
        C.zero_()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):  # warm-up on the capture stream: its workspace exists before capture
            tsm.gemm(A, B, C, variant=variant, c_is_zero=True)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            tsm.gemm(A, B, C, variant=variant, c_is_zero=True)
        ref = naive_gemm(A.cpu().numpy(), B.cpu().numpy(), np.zeros((m, n), A.cpu().numpy().dtype))
        for _ in range(3):
            C.fill_(123.0)
            g.replay()
            torch.cuda.synchronize()
            prec = "double" if dt == torch.float64 else "single"
            assert rel_frobenius(C.cpu().numpy(), ref) <= TOL_FROB[prec], (m, k, n, dt)


@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("m,k,n,c_zero", [(100003, 16, 16, True), (4099, 7, 8, False), (65536, 64, 4, False),
                                         (333, 16, 5, True), (1, 3, 16, False)])
def test_tsm2l_splitn_against_oracle(prec, m, k, n, c_zero):
    """The split-n warp-shuffle TSM2L kernel (impl tsm2l-splitn): ragged m, k not a multiple of
    the 4-way split, pass widths 4/8/16 and a ragged last pass, zero and nonzero C."""
    import torch
    from oracle.rng import uniform_block
    tsm = _tsm()
    dt = torch.float64 if prec == "double" else torch.float32
    npdt = np.float64 if prec == "double" else np.float32
    A = tsm.colmajor_empty(m, k, dt, "cuda")
    tsm.fill_uniform(A, seed=61)
    B = tsm.colmajor_empty(k, n, dt, "cuda")
    tsm.fill_uniform(B, seed=62)
    C = tsm.colmajor_empty(m, n, dt, "cuda")
    if c_zero:
        C.fill_(float("nan"))
    else:
        tsm.fill_uniform(C, seed=63)
    C0h = np.zeros((m, n), npdt) if c_zero else C.cpu().numpy()
    tsm.gemm(A, B, C, variant="l-opt2" if c_zero else "l-opt1", c_is_zero=c_zero, impl="tsm2l-splitn")
    torch.cuda.synchronize()
    ref = naive_gemm(uniform_block(range(m), range(k), 61).astype(npdt), uniform_block(range(k), range(n), 62).astype(npdt),
                     C0h)
    _check(C.cpu().numpy(), ref, k, prec, what=("splitn", m, k, n, c_zero))


def test_fp32_small_direct_reductions():
    """Small fp32 C += calls (A <= 128 MB) run as one FFMA2 launch whose split row blocks reduce in
    fp32 straight into C (no fp64 accumulator, no finalize): C += A.B within the fp32 tolerance on
    even, ragged and equal-split shapes, and C's prior contents are kept."""
    import torch
    tsm = _tsm()
    from paper_2002_03258_b200 import tuning
    rng = np.random.default_rng(23)
    for (m, k, n) in [(512, 512, 16), (1024, 1024, 16), (4096, 4096, 16), (1000, 3000, 13), (2048, 5000, 8),
                      (300, 20000, 16)]:
        assert tuning.plan("single", m, k, n)["consumer"] == "ffma2", (m, k, n)
        A = tsm.colmajor_empty(m, k, torch.float32, "cuda")
        A.copy_(torch.from_numpy(rng.random((m, k)).astype(np.float32)))
        B = tsm.colmajor_empty(k, n, torch.float32, "cuda")
        B.copy_(torch.from_numpy(rng.random((k, n)).astype(np.float32)))
        C0 = rng.random((m, n)).astype(np.float32) * 100
        C = tsm.colmajor_empty(m, n, torch.float32, "cuda")
        C.copy_(torch.from_numpy(C0))
        tsm.gemm(A, B, C)
        ref = C0.astype(np.float64) + A.cpu().numpy().astype(np.float64) @ B.cpu().numpy().astype(np.float64)
        assert rel_frobenius(C.cpu().numpy().astype(np.float64), ref) <= 1e-5, (m, k, n)
