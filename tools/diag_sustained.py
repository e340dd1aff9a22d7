"""Diagnostic build only: per-stage cycle counters of the stream kernel's consumer loop while the
part runs back to back (power-capped) — are the consumers waiting for data (memory-bound) or is
the data waiting for them (consumer-bound)?  TSM2X_LIB_PATH_EXPERIMENT=...libtsm2x_diag.so
TSM2X_TC_DIAG=0 python tools/diag_sustained.py r8"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_03258_b200 as tsm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "r8"
m, k, n = {"r8": (30720, 30720, 8), "r16": (30720, 30720, 16)}[cfg]
A = tsm.colmajor_empty(m, k, torch.float64, "cuda"); tsm.fill_uniform(A, 1)
B = tsm.colmajor_empty(k, n, torch.float64, "cuda"); tsm.fill_uniform(B, 2)
C = tsm.colmajor_empty(m, n, torch.float64, "cuda"); C.zero_()
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 600):
    tsm.gemm(A, B, C)  # the diagnostic build syncs and prints one line per call (stderr)
