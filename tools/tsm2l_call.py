"""One TSM2L shape called 30 times (for ncu): python tools/tsm2l_call.py f|d [impl] [n] [k] [m_log2]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2002_03258_b200 as tsm  # noqa: E402

dt = torch.float32 if sys.argv[1] == "f" else torch.float64
impl = sys.argv[2] if len(sys.argv) > 2 else "auto"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 16
k = int(sys.argv[4]) if len(sys.argv) > 4 else 16
m = 1 << (int(sys.argv[5]) if len(sys.argv) > 5 else 24)
A = tsm.colmajor_empty(m, k, dt, "cuda"); tsm.fill_uniform(A, 1)
B = tsm.colmajor_empty(k, n, dt, "cuda"); tsm.fill_uniform(B, 2)
C = tsm.colmajor_empty(m, n, dt, "cuda"); C.zero_()
for _ in range(30):
    tsm.gemm(A, B, C, variant="l-opt2", c_is_zero=True, impl=impl)
torch.cuda.synchronize()
