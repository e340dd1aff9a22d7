"""Boundary types of the drop-in: Precision, Variant, Matrix, KernelParams, ShapeClass.

These mirror the argument conventions of the reference package so a caller of
``tsgemm.run_native`` can switch imports and keep its code:

* ``Precision``  — reference ``pkg/src/tsgemm/core.py:23-46``
* ``ShapeClass`` / ``validate_problem`` — ``core.py:49-54, 297-313``
* ``Variant``    — ``core.py:57-81`` (same values, ``parse``, ``uses_shared_tile``, ``is_tsm2l``)
* ``Matrix``     — ``core.py:84-157``: dense column-major, element (i, j) at flat index
  ``i + j * rows``, frozen backing store, "modifying" operations return new matrices
* ``KernelParams`` — ``core.py:160-190``: the (t1, t2, t3, tcf) tuple with the same
  constructor invariants and ``validate_for`` rules, raising ``ValueError`` with the same
  conditions.

Reference objects are accepted wherever these are (duck typing on ``rows``, ``cols``,
``storage``, ``precision.value`` and on ``t1..tcf``/``variant.value``), so matrices built
with the reference package can be passed straight to :func:`run_native`.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

WARP_SIZE = 32


class Precision(enum.Enum):
    SINGLE = "single"
    DOUBLE = "double"

    @property
    def bytes_per_element(self) -> int:
        return 8 if self is Precision.DOUBLE else 4

    @property
    def dtype(self) -> np.dtype:
        return np.dtype(np.float64) if self is Precision.DOUBLE else np.dtype(np.float32)

    @property
    def eps(self) -> float:
        return float(np.finfo(self.dtype).eps)

    @classmethod
    def parse(cls, text: str) -> "Precision":
        key = str(text).lower()
        for p in cls:
            if p.value == key:
                return p
        raise ValueError(f"unknown precision {text!r}; expected 'single' or 'double'")

    @classmethod
    def coerce(cls, obj) -> "Precision":
        """Accepts our enum, the reference enum (same ``.value``), or a string."""
        if isinstance(obj, cls):
            return obj
        return cls.parse(getattr(obj, "value", obj))


class ShapeClass(enum.Enum):
    TSM2R = "tsm2r"
    TSM2L = "tsm2l"
    GENERAL = "general"


DOMINANCE_FACTOR = 16


def validate_problem(m: int, k: int, n: int, variant=None) -> ShapeClass:
    """Advisory (m, k, n) classification; raises only for non-positive dimensions."""
    for name, d in (("m", m), ("k", k), ("n", n)):
        if d < 1:
            raise ValueError(f"dimension {name} must be >= 1, got {d}")
    f = DOMINANCE_FACTOR
    big, small = max(m, k), min(m, k)
    if big <= f * small and small >= f * n:
        return ShapeClass.TSM2R
    if m >= f * max(k, n) and max(k, n) <= f * min(k, n):
        return ShapeClass.TSM2L
    return ShapeClass.GENERAL


class Variant(enum.Enum):
    V0 = "v0"
    V1 = "v1"
    V2 = "v2"
    V3 = "v3"
    L_OPT1 = "l-opt1"
    L_OPT2 = "l-opt2"

    @classmethod
    def parse(cls, text: str) -> "Variant":
        key = str(text).lower().replace("_", "-")
        for v in cls:
            if v.value == key:
                return v
        raise ValueError(f"unknown kernel variant {text!r}")

    @classmethod
    def coerce(cls, obj) -> "Variant":
        if isinstance(obj, cls):
            return obj
        return cls.parse(getattr(obj, "value", obj))

    @property
    def ordinal(self) -> int:
        """Index used by the C ABI (include/tsm2x.h enum tsm2x_variant)."""
        return list(Variant).index(self)

    @property
    def uses_shared_tile(self) -> bool:
        return self in (Variant.V2, Variant.V3, Variant.L_OPT1, Variant.L_OPT2)

    @property
    def is_tsm2l(self) -> bool:
        return self in (Variant.L_OPT1, Variant.L_OPT2)


_PAR_COPY_BYTES = 64 << 20


def _copy_flat(storage, dtype) -> np.ndarray:
    """A private flat copy of ``storage`` (the reference's Matrix copies its input, core.py:101).
    Large contiguous arrays are copied in parallel slices (numpy releases the GIL in copyto), so
    building a 7.5 GB Matrix is bound by memory bandwidth rather than one core."""
    src = np.asarray(storage)
    if src.dtype != dtype or src.nbytes < _PAR_COPY_BYTES or not src.flags.c_contiguous:
        return np.array(src, dtype=dtype, copy=True).reshape(-1)
    src = src.reshape(-1)
    out = np.empty(src.size, dtype=dtype)
    import os
    from concurrent.futures import ThreadPoolExecutor
    nt = max(1, min(16, os.cpu_count() or 1))
    cuts = [src.size * i // nt for i in range(nt + 1)]
    with ThreadPoolExecutor(nt) as pool:
        list(pool.map(lambda i: np.copyto(out[cuts[i]:cuts[i + 1]], src[cuts[i]:cuts[i + 1]]), range(nt)))
    return out


class Matrix:
    """Dense column-major matrix over a frozen flat numpy array (element (i, j) at i + j*rows)."""

    __slots__ = ("rows", "cols", "storage", "precision")

    def __init__(self, rows: int, cols: int, storage, precision: Precision):
        precision = Precision.coerce(precision)
        if rows < 1 or cols < 1:
            raise ValueError(f"matrix dimensions must be positive, got {rows}x{cols}")
        flat = _copy_flat(storage, precision.dtype)
        if flat.size != rows * cols:
            raise ValueError(f"storage length {flat.size} != rows*cols = {rows * cols}")
        flat.flags.writeable = False
        self.rows, self.cols, self.storage, self.precision = rows, cols, flat, precision

    @classmethod
    def _adopt(cls, rows: int, cols: int, flat: np.ndarray, precision: Precision) -> "Matrix":
        """Wraps a freshly produced array without another copy (internal: results of run_native)."""
        obj = cls.__new__(cls)
        flat = flat.reshape(-1)
        flat.flags.writeable = False
        obj.rows, obj.cols, obj.storage, obj.precision = rows, cols, flat, precision
        return obj

    @classmethod
    def zeros(cls, rows: int, cols: int, precision: Precision) -> "Matrix":
        precision = Precision.coerce(precision)
        if rows < 1 or cols < 1:
            raise ValueError(f"matrix dimensions must be positive, got {rows}x{cols}")
        return cls._adopt(rows, cols, np.zeros(rows * cols, dtype=precision.dtype), precision)

    @classmethod
    def from_2d(cls, array, precision: Precision) -> "Matrix":
        precision = Precision.coerce(precision)
        arr = np.asarray(array, dtype=precision.dtype)
        if arr.ndim != 2:
            raise ValueError("expected a 2-D array")
        return cls(arr.shape[0], arr.shape[1], arr.reshape(-1, order="F"), precision)

    @classmethod
    def random(cls, rows: int, cols: int, precision: Precision, rng: np.random.Generator) -> "Matrix":
        """Uniform [0, 1): float64 draws cast to the precision (reference core.py:119-123)."""
        precision = Precision.coerce(precision)
        draws = rng.random(rows * cols, dtype=np.float64).astype(precision.dtype)
        return cls(rows, cols, draws, precision)

    @classmethod
    def identity(cls, n: int, precision: Precision) -> "Matrix":
        precision = Precision.coerce(precision)
        return cls.from_2d(np.eye(n, dtype=precision.dtype), precision)

    def _check(self, i: int, j: int) -> None:
        if not (0 <= i < self.rows and 0 <= j < self.cols):
            raise IndexError(f"({i}, {j}) out of bounds for {self.rows}x{self.cols}")

    def get(self, i: int, j: int) -> float:
        self._check(i, j)
        return float(self.storage[i + j * self.rows])

    def with_element(self, i: int, j: int, value: float) -> "Matrix":
        self._check(i, j)
        data = self.storage.copy()
        data[i + j * self.rows] = value
        return Matrix(self.rows, self.cols, data, self.precision)

    def column(self, j: int) -> np.ndarray:
        return self.storage[j * self.rows:(j + 1) * self.rows]

    def to_2d(self) -> np.ndarray:
        return self.storage.reshape((self.rows, self.cols), order="F")

    def __eq__(self, other) -> bool:
        """Equal to any Matrix-like object (this class or the reference's) with the same shape,
        precision and storage bits."""
        try:
            rows, cols, storage = other.rows, other.cols, other.storage
            prec = Precision.coerce(other.precision)
        except (AttributeError, ValueError):
            return False
        return (self.rows, self.cols, self.precision) == (rows, cols, prec) and bool(
            np.array_equal(self.storage, storage))

    __hash__ = None

    def __repr__(self) -> str:
        return f"Matrix({self.rows}x{self.cols}, {self.precision.value})"


def result_like(C, rows: int, cols: int, flat: np.ndarray, precision: Precision):
    """The result Matrix of run_native, of the caller's Matrix type: when C is a reference
    ``tsgemm.Matrix`` (same ``__slots__`` layout, reference core.py:84-106) the result is one too,
    so ``==`` against reference results (whose ``__eq__`` checks ``isinstance``) keeps working.
    The freshly produced array is adopted without a copy either way."""
    cls = type(C)
    # only a Matrix class proper (the reference's: same __slots__ and methods) is mirrored; other
    # duck-typed inputs get this package's Matrix
    if cls is Matrix or tuple(getattr(cls, "__slots__", ())) != Matrix.__slots__ or not hasattr(cls, "to_2d"):
        return Matrix._adopt(rows, cols, flat, precision)
    obj = cls.__new__(cls)
    flat = flat.reshape(-1)
    flat.flags.writeable = False
    obj.rows, obj.cols, obj.storage = rows, cols, flat
    obj.precision = C.precision  # the caller's Precision enum member
    return obj


@dataclass(frozen=True)
class KernelParams:
    """(t1, t2, t3, tcf): threads per block / B-tile rows, C columns per pass, A elements per
    prefetch, row tiles per thread (TSM2L). Same invariants as the reference (core.py:176-190).

    On B200 these are validated exactly as the reference does and drive the paper's V0/V1/V2
    ablation kernels; the production V3 / L_OPT1 / L_OPT2 kernels take their tiling from the
    B200 table in :mod:`paper_2002_03258_b200.tuning` (results never depend on params,
    as in the reference, README.md:88-92).
    """

    t1: int = 128
    t2: int = 4
    t3: int = 4
    tcf: int = 1
    variant: Variant = Variant.V3

    def __post_init__(self):
        for name in ("t1", "t2", "t3", "tcf"):
            value = getattr(self, name)
            if value < 1:
                raise ValueError(f"{name} must be >= 1, got {value}")
        if self.t3 > self.t1:
            raise ValueError(f"t3 ({self.t3}) must not exceed t1 ({self.t1})")

    def validate_for(self, m: int, k: int, n: int, warp_size: int = WARP_SIZE) -> None:
        validate_params_for(self, m, k, n, warp_size)


def validate_params_for(params, m: int, k: int, n: int, warp_size: int = WARP_SIZE) -> None:
    """The reference's ``KernelParams.validate_for`` rules on any params-like object."""
    if params.t2 > n:
        raise ValueError(f"t2 ({params.t2}) must not exceed n ({n})")
    if params.t1 % warp_size != 0:
        raise ValueError(f"t1 ({params.t1}) must be a multiple of warp size {warp_size}")
    if params.tcf > 1 and not Variant.coerce(params.variant).is_tsm2l:
        raise ValueError("tcf > 1 is only meaningful for the TSM2L variants")


def check_dims(A, B, C) -> tuple:
    """Reference ``kernels._check_dims`` (kernels.py:36-44): returns (m, k, n)."""
    if A.cols != B.rows or A.rows != C.rows or B.cols != C.cols:
        raise ValueError(
            f"dimension mismatch: A {A.rows}x{A.cols}, B {B.rows}x{B.cols}, C {C.rows}x{C.cols}")
    pa, pb, pc = (Precision.coerce(X.precision) for X in (A, B, C))
    if not (pa is pb is pc):
        raise ValueError("A, B, C must share one precision")
    return A.rows, A.cols, B.cols
