"""B200-native TSM2X (arXiv 2002.03258): TSM2R / TSM2L tall-and-skinny GEMM on sm_100a.

Drop-in for the reference package's hot path (``tsgemm.run_native`` and its boundary types,
reference ``pkg/src/tsgemm/__init__.py:9-22``) over ``libtsm2x.so`` (C ABI: include/tsm2x.h).
"""

from .core import (  # noqa: F401
    KernelParams,
    Matrix,
    Precision,
    ShapeClass,
    Variant,
    validate_problem,
)
from .kernels import (  # noqa: F401
    colmajor_empty,
    fill_uniform,
    gemm,
    gemm_multi,
    release_cached_memory,
    run_native,
    row_range,
    run_native_multi,
    simulate,
)

__all__ = [
    "KernelParams",
    "Matrix",
    "Precision",
    "ShapeClass",
    "Variant",
    "colmajor_empty",
    "fill_uniform",
    "gemm",
    "gemm_multi",
    "release_cached_memory",
    "run_native",
    "row_range",
    "run_native_multi",
    "simulate",
    "validate_problem",
]

__version__ = "0.1.0"
