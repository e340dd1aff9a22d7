"""Counter-based U[0,1) generator, bit-identical to the CUDA ``tsm2x_fill_uniform`` kernel
(include/tsm2x.h) — test infrastructure for regenerating any row slab of the large synthetic
inputs (configs 2-5) on the host without materialising the whole matrix.

  x = splitmix64(seed * 0x9E3779B97F4A7C15 + ((col << 32) | row))     (uint64, wrapping)
  u = (x >> 11) * 2**-53                                             (float64 in [0, 1))
  float32 inputs use u.astype(float32), as Matrix.random does (reference core.py:119-123).
"""

from __future__ import annotations

import numpy as np

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + _GOLD
        x = (x ^ (x >> np.uint64(30))) * _M1
        x = (x ^ (x >> np.uint64(27))) * _M2
        return x ^ (x >> np.uint64(31))


def uniform_block(rows, cols, seed: int, dtype=np.float64) -> np.ndarray:
    """Values at global positions (rows[i], cols[j]) as a 2-D (len(rows), len(cols)) F-array.

    ``rows``/``cols`` are integer sequences or ranges of global indices.
    """
    r = np.asarray(rows, dtype=np.uint64).reshape(-1, 1)
    c = np.asarray(cols, dtype=np.uint64).reshape(1, -1)
    with np.errstate(over="ignore"):
        base = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) * _GOLD
        key = (c << np.uint64(32)) | r
        x = _splitmix64(base + key)
    u = (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return np.asfortranarray(u.astype(dtype))
