"""CPU oracle for the TSM2R/TSM2L hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the reference's arithmetic for the path so the CUDA kernels
can be checked against it. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline leg (``cpu_baseline`` / ``--impl reference``) may import it, and only as the checker
or the timed CPU arm — never as part of the shipped product (``paper_2002_03258_b200`` does
not import it and has no CPU fallback).

Parity pinning: the restatement is checked bit-for-bit against outputs produced by the
reference package itself (``/root/reference/pkg/src/tsgemm``, imported in the build container
by ``tests/golden/make_golden.py``) and committed as ``tests/golden/golden.json`` +
``golden.npz``. See DESIGN.md §3.

Modules:
  reference  naive_gemm / max_rel_error (reference oracle.py:19-45) and the reference's
             vectorised run_native body (kernels.py:391-416), plus row-slab and threaded forms
  rng        the counter-based U[0,1) generator shared with the CUDA fill kernel
"""

from .reference import (  # noqa: F401
    max_rel_error,
    naive_gemm,
    naive_gemm_rows,
    rel_frobenius,
    run_native_port,
    run_native_port_threaded,
)
from .rng import uniform_block  # noqa: F401
