"""numpy restatement of the reference's arithmetic on the hot path (test infrastructure).

Arrays here are plain 2-D numpy arrays (m x k, k x n, m x n); any memory order.

* :func:`naive_gemm` follows reference ``pkg/src/tsgemm/oracle.py:19-37``: accumulate
  ``C0 + sum_l A[:, l] * B[l, :]`` over ascending l in float64 (also for float32 inputs), round
  once to the input precision.
* :func:`run_native_port` follows reference ``pkg/src/tsgemm/kernels.py:391-416``: for each
  pass of t2 columns, for ascending e, an unfused multiply rounded to the input precision then
  an add rounded to the input precision (two numpy ufunc passes), starting from C.
  For float64 it is bitwise equal to ``naive_gemm`` (same order, same rounding), which the
  golden fixtures confirm.
* :func:`max_rel_error` follows reference ``oracle.py:40-45``.
* :func:`rel_frobenius` is the BASELINE.json parity metric (||R - E||_F / ||E||_F).

Rows are independent, so a row slab computed alone is bitwise identical to the same rows of
the full product (:func:`naive_gemm_rows`, :func:`run_native_port_threaded`).
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np


def naive_gemm(A: np.ndarray, B: np.ndarray, C0: np.ndarray) -> np.ndarray:
    if A.shape[1] != B.shape[0] or A.shape[0] != C0.shape[0] or B.shape[1] != C0.shape[1]:
        raise ValueError(f"dimension mismatch: A {A.shape}, B {B.shape}, C0 {C0.shape}")
    out_dtype = A.dtype
    acc = np.array(C0, dtype=np.float64, order="F", copy=True)
    Af = A.astype(np.float64, copy=False)
    Bf = B.astype(np.float64, copy=False)
    for l in range(A.shape[1]):
        acc += Af[:, l:l + 1] * Bf[l:l + 1, :]
    return acc.astype(out_dtype)


def naive_gemm_rows(A: np.ndarray, B: np.ndarray, C0: np.ndarray, rows) -> np.ndarray:
    """naive_gemm restricted to a subset/slab of rows (bitwise equal to those rows of the full)."""
    return naive_gemm(A[rows], B, C0[rows])


def run_native_port(A: np.ndarray, B: np.ndarray, C: np.ndarray, t2: int | None = None) -> np.ndarray:
    m, k = A.shape
    n = B.shape[1]
    t2 = n if t2 is None else t2
    out = np.array(C, dtype=A.dtype, order="F", copy=True)
    for p in range(0, n, t2):
        w = min(t2, n - p)
        acc = out[:, p:p + w].copy()
        tmp = np.empty_like(acc)
        for e in range(k):
            np.multiply(A[:, e:e + 1], B[e:e + 1, p:p + w], out=tmp)
            np.add(acc, tmp, out=acc)
        out[:, p:p + w] = acc
    return out


def run_native_port_threaded(A: np.ndarray, B: np.ndarray, C: np.ndarray, threads: int | None = None,
                             t2: int | None = None) -> np.ndarray:
    """run_native_port over row slabs on a thread pool (numpy ufuncs release the GIL).

    Bitwise equal to the single-threaded port; this is how the reference's CPU path is given
    all host cores for the benchmark's reference arm.
    """
    threads = threads or len(os.sched_getaffinity(0))
    m = A.shape[0]
    out = np.empty((m, B.shape[1]), dtype=A.dtype, order="F")
    bounds = np.linspace(0, m, threads + 1).astype(int)

    def work(i):
        lo, hi = bounds[i], bounds[i + 1]
        if hi > lo:
            out[lo:hi] = run_native_port(A[lo:hi], B, C[lo:hi], t2)

    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(work, range(threads)))
    return out


def max_rel_error(result: np.ndarray, reference: np.ndarray) -> float:
    r = np.asarray(result, dtype=np.float64)
    e = np.asarray(reference, dtype=np.float64)
    return float(np.max(np.abs(r - e) / np.maximum(np.abs(e), 1.0)))


def rel_frobenius(result: np.ndarray, reference: np.ndarray) -> float:
    r = np.asarray(result, dtype=np.float64)
    e = np.asarray(reference, dtype=np.float64)
    den = float(np.linalg.norm(e))
    num = float(np.linalg.norm(r - e))
    return num / den if den > 0 else num
