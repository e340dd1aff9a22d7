"""The drop-in entry points.

* :func:`run_native` — same signature, argument conventions and errors as the reference
  ``tsgemm.kernels.run_native(variant, A, B, C, params) -> Matrix`` (kernels.py:391-416):
  returns a NEW frozen Matrix holding ``C + A @ B`` (the caller's C is never mutated); L_OPT2
  requires an all-zero C (kernels.py:366-368). Host matrices go through ``tsm2x_run_host``,
  which pipelines the H2D copy of A with the sm_100a kernels.
* :func:`gemm` — the device-resident form on column-major torch CUDA tensors
  (``tsm2x_run``), stream-ordered, for callers that keep A in HBM (the benchmark, the
  multi-GPU driver, k-means / ABFT consumers named in PAPER.md:55-56).
* :func:`simulate` — the reference's SIMT-simulator entry point has no GPU meaning; it raises
  NotImplementedError pointing at ncu (out of scope).

Results never depend on ``params`` (reference README.md:88-92); the production kernels take
their tiling from :mod:`paper_2002_03258_b200.tuning`.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .core import Matrix, Precision, Variant, check_dims, result_like, validate_params_for


def _params_struct(params) -> _lib.Params:
    v = Variant.coerce(getattr(params, "variant", Variant.V3))
    return _lib.Params(int(params.t1), int(params.t2), int(params.t3), int(params.tcf), v.ordinal)


def _flat(M, dtype) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(M.storage).reshape(-1))
    if a.dtype != dtype:
        a = a.astype(dtype)
    return a


def _host_call(variant, A, B, C, params, deterministic):
    """Validation + host arrays shared by run_native / run_native_multi."""
    variant = Variant.coerce(variant)
    m, k, n = check_dims(A, B, C)
    validate_params_for(params, m, k, n)
    prec = Precision.coerce(A.precision)
    dtype = prec.dtype
    a, b, c = _flat(A, dtype), _flat(B, dtype), _flat(C, dtype)
    # L_OPT2's zero-C rule (reference kernels.py:366-368) is checked by tsm2x_run_host on the host
    # copy — a parallel scan with early exit, before any device work — and raises the same
    # ValueError through _lib.check
    flags = _lib.FLAG_DETERMINISTIC if deterministic else 0
    return variant, m, k, n, prec, a, b, c, flags


def run_native(variant, A, B, C, params, *, deterministic: bool = True) -> Matrix:
    """``C + A @ B`` on the B200 for column-major Matrix inputs (reference kernels.py:391-416).

    ``deterministic`` (default on): split row blocks combine in column order, so repeated calls
    return the same bits, as the reference's do. The host path is bound by the PCIe copy of A,
    so the ordered combine costs nothing measurable here (it is 5-30 % of the kernel alone).
    The result has the caller's Matrix type (reference Matrix in, reference Matrix out).
    """
    variant, m, k, n, prec, a, b, c, flags = _host_call(variant, A, B, C, params, deterministic)
    out = np.empty(m * n, dtype=prec.dtype)
    lib = _lib.load()
    p = _params_struct(params)
    rc = lib.tsm2x_run_host(
        variant.ordinal, _lib.DOUBLE if prec is Precision.DOUBLE else _lib.SINGLE, m, k, n,
        a.ctypes.data, m, b.ctypes.data, k, c.ctypes.data, out.ctypes.data, m, ctypes.byref(p), flags,
        _current_device())
    _lib.check(rc)
    return result_like(C, m, n, out, prec)


def run_native_multi(variant, A, B, C, params, devices, *, deterministic: bool = True) -> Matrix:
    """run_native over several GPUs of this process (``tsm2x_run_host_multi``): contiguous
    32-row-aligned row shards, one per entry of ``devices`` (may repeat), each streamed by its
    own host thread, so the per-GPU PCIe links add up. Same result contract as run_native."""
    variant, m, k, n, prec, a, b, c, flags = _host_call(variant, A, B, C, params, deterministic)
    devices = list(devices)
    if not devices:
        raise ValueError("devices must not be empty")
    devs = (ctypes.c_int * len(devices))(*devices)
    out = np.empty(m * n, dtype=prec.dtype)
    p = _params_struct(params)
    rc = _lib.load().tsm2x_run_host_multi(
        variant.ordinal, _lib.DOUBLE if prec is Precision.DOUBLE else _lib.SINGLE, m, k, n, a.ctypes.data, m,
        b.ctypes.data, k, c.ctypes.data, out.ctypes.data, m, ctypes.byref(p), flags, len(devices), devs)
    _lib.check(rc)
    return result_like(C, m, n, out, prec)


def simulate(*args, **kwargs):
    raise NotImplementedError(
        "simulate() is the reference's CPU SIMT model (kernels.py:371-388); on B200 the real kernels run "
        "via run_native/gemm and Nsight Compute supplies the counters (see DESIGN.md)")


def _current_device() -> int:
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # pragma: no cover - torch absent
        pass
    return 0


# ---------------------------------------------------------------------------------------------
# device-resident API (torch tensors)

def colmajor_empty(rows: int, cols: int, dtype, device, pad_to: int = 32):
    """An uninitialised (rows x cols) column-major CUDA tensor whose leading dimension is
    padded to a multiple of ``pad_to`` elements (keeps every column 16-B aligned for TMA)."""
    import torch
    ld = (rows + pad_to - 1) // pad_to * pad_to
    base = torch.empty((cols, ld), dtype=dtype, device=device)
    return base.t()[:rows, :]


def _ld(t, rows: int) -> int:
    """Leading dimension of a column-major tensor. Layouts whose columns overlap (stride(1) <
    rows, e.g. expand() or a stride-0 broadcast) are rejected: the kernels would read past the
    storage or write aliased elements."""
    if t.dim() != 2:
        raise ValueError("expected a 2-D tensor")
    s0, s1 = t.stride()
    if s0 != 1 and not (t.shape[0] == 1):
        raise ValueError("tensor must be column-major (stride(0) == 1); use colmajor_empty or x.t().contiguous().t()")
    if t.shape[1] == 1:
        return max(int(s1), rows)  # one column: its stride is never used
    if s1 < rows:
        raise ValueError(f"column stride {s1} < rows {rows}: overlapping columns (expanded or broadcast tensor); "
                         "pass a dense column-major tensor")
    return int(s1)


def gemm(A, B, C, *, variant=Variant.V3, params=None, c_is_zero: bool = False, impl: str = "auto",
         stream=None, check_zero_c: bool = False, deterministic: bool = False):
    """In place on device: ``C (+)= A @ B`` for column-major CUDA tensors (fp32 or fp64).

    ``c_is_zero`` elides the read of C (the L_OPT2 contract). ``deterministic`` makes the result
    bitwise reproducible run to run: row blocks split across CTAs are then combined in column
    order through per-row-block tickets instead of with fp64 atomics (same tolerance either way;
    the atomic default is faster).
    Stream-ordered on ``stream`` (default: torch's current stream); returns C.
    """
    import torch
    from .core import KernelParams
    variant = Variant.coerce(variant)
    if not (A.is_cuda and B.is_cuda and C.is_cuda):
        raise ValueError("gemm expects CUDA tensors; use run_native for host matrices")
    if not (A.dtype == B.dtype == C.dtype) or A.dtype not in (torch.float32, torch.float64):
        raise ValueError("A, B, C must share one precision (float32 or float64)")
    m, k = A.shape
    if B.shape[0] != k or C.shape[0] != m or B.shape[1] != C.shape[1]:
        raise ValueError(f"dimension mismatch: A {m}x{k}, B {B.shape[0]}x{B.shape[1]}, C {C.shape[0]}x{C.shape[1]}")
    n = B.shape[1]
    if params is None:
        params = KernelParams(t1=128, t2=min(4, n), t3=4, tcf=1, variant=variant)
    validate_params_for(params, m, k, n)
    prec = _lib.DOUBLE if A.dtype == torch.float64 else _lib.SINGLE
    flags = (_lib.FLAG_C_IS_ZERO if c_is_zero else 0) | (_lib.FLAG_CHECK_ZERO_C if check_zero_c else 0) | \
        (_lib.FLAG_DETERMINISTIC if deterministic else 0)
    if stream is None:
        stream = torch.cuda.current_stream(A.device)
    p = _params_struct(params)
    with torch.cuda.device(A.device):
        rc = _lib.load().tsm2x_run_ex(
            variant.ordinal, prec, m, k, n, A.data_ptr(), _ld(A, m), B.data_ptr(), _ld(B, k), C.data_ptr(),
            _ld(C, m), ctypes.byref(p), flags, _lib.IMPL[impl], ctypes.c_void_p(stream.cuda_stream))
    _lib.check(rc)
    return C


def row_range(m: int, ndev: int, g: int):
    """Rows [r0, r1) of shard ``g`` of an m-row problem over ``ndev`` shards (``tsm2x_row_range``:
    contiguous, balanced in 32-row units — the same split as ``multi.row_partition``)."""
    r0, r1 = ctypes.c_int64(), ctypes.c_int64()
    _lib.load().tsm2x_row_range(int(m), int(ndev), int(g), ctypes.byref(r0), ctypes.byref(r1))
    return r0.value, r1.value


def gemm_multi(A_shards, B, C_shards, *, variant=Variant.V3, params=None, c_is_zero: bool = False,
               deterministic: bool = False, streams=None):
    """``gemm`` over several GPUs of this process (``tsm2x_run_multi``): ``A_shards[g]`` /
    ``C_shards[g]`` are the rows ``row_range(m, len(A_shards), g)`` of A / C as column-major CUDA
    tensors on their own devices (devices may repeat), B lives on ``A_shards[0]``'s device and
    is copied to the other devices over NVLink inside the call; every shard is stream-ordered on
    ``streams[g]`` (default: torch's current stream of its device). No reduction — rows are
    independent (reference SPEC.md:262). Returns ``C_shards``."""
    import torch
    from .core import KernelParams
    variant = Variant.coerce(variant)
    nd = len(A_shards)
    if nd < 1 or len(C_shards) != nd:
        raise ValueError("need one A shard and one C shard per device")
    dt = B.dtype
    if dt not in (torch.float32, torch.float64) or any(t.dtype != dt for t in list(A_shards) + list(C_shards)):
        raise ValueError("A, B, C must share one precision (float32 or float64)")
    if not all(t.is_cuda for t in list(A_shards) + list(C_shards) + [B]):
        raise ValueError("gemm_multi expects CUDA tensors")
    k, n = B.shape
    m = sum(int(a.shape[0]) for a in A_shards)
    for g, (a, c) in enumerate(zip(A_shards, C_shards)):
        r0, r1 = row_range(m, nd, g)
        if a.shape != (r1 - r0, k) or c.shape != (r1 - r0, n) or a.device != c.device:
            raise ValueError(f"shard {g}: expected A {r1 - r0}x{k} and C {r1 - r0}x{n} on one device "
                             f"(rows {r0}:{r1} of {m}), got A {tuple(a.shape)} on {a.device}, "
                             f"C {tuple(c.shape)} on {c.device}")
    if B.device != A_shards[0].device:
        raise ValueError("B must live on the first shard's device")
    if params is None:
        params = KernelParams(t1=128, t2=min(4, n), t3=4, tcf=1, variant=variant)
    validate_params_for(params, m, k, n)
    prec = _lib.DOUBLE if dt == torch.float64 else _lib.SINGLE
    flags = (_lib.FLAG_C_IS_ZERO if c_is_zero else 0) | (_lib.FLAG_DETERMINISTIC if deterministic else 0)
    if streams is None:
        streams = [torch.cuda.current_stream(a.device) for a in A_shards]
    i64 = ctypes.c_int64
    devs = (ctypes.c_int * nd)(*[a.device.index for a in A_shards])
    a_ptr = (ctypes.c_void_p * nd)(*[a.data_ptr() for a in A_shards])
    c_ptr = (ctypes.c_void_p * nd)(*[c.data_ptr() for c in C_shards])
    lda = (i64 * nd)(*[_ld(a, a.shape[0]) if a.shape[0] else 1 for a in A_shards])
    ldc = (i64 * nd)(*[_ld(c, c.shape[0]) if c.shape[0] else 1 for c in C_shards])
    st = (ctypes.c_void_p * nd)(*[s.cuda_stream for s in streams])
    p = _params_struct(params)
    rc = _lib.load().tsm2x_run_multi(variant.ordinal, prec, m, k, n, nd, devs, a_ptr, lda, B.data_ptr(), _ld(B, k),
                                     c_ptr, ldc, ctypes.byref(p), flags, st)
    _lib.check(rc)
    return C_shards


def fill_uniform(T, seed: int, row_offset: int = 0, col_offset: int = 0, stream=None):
    """Fills a column-major CUDA tensor with the counter-based U[0,1) generator (tsm2x.h)."""
    import torch
    rows, cols = T.shape
    prec = _lib.DOUBLE if T.dtype == torch.float64 else _lib.SINGLE
    if stream is None:
        stream = torch.cuda.current_stream(T.device)
    with torch.cuda.device(T.device):
        rc = _lib.load().tsm2x_fill_uniform(prec, rows, cols, T.data_ptr(), _ld(T, rows), row_offset, col_offset,
                                            seed & 0xFFFFFFFFFFFFFFFF, ctypes.c_void_p(stream.cuda_stream))
    _lib.check(rc)
    return T


def release_cached_memory(device: int = -1) -> None:
    """Frees the library's cached device / pinned memory (per-stream workspaces, host-path staging)
    on ``device`` (-1: all devices) after synchronising it (``tsm2x_release_cached``). For
    long-lived processes that create many streams; later calls re-allocate what they need."""
    _lib.check(_lib.load().tsm2x_release_cached(int(device)))
