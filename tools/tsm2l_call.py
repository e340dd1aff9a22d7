import sys, torch
sys.path.insert(0, ".")
import paper_2002_03258_b200 as tsm
m, k, n = 1 << 24, 16, 16
dt = torch.float32 if sys.argv[1] == "f" else torch.float64
A = tsm.colmajor_empty(m, k, dt, "cuda"); tsm.fill_uniform(A, 1)
B = tsm.colmajor_empty(k, n, dt, "cuda"); tsm.fill_uniform(B, 2)
C = tsm.colmajor_empty(m, n, dt, "cuda"); C.zero_()
for _ in range(30):
    tsm.gemm(A, B, C, variant="l-opt2", c_is_zero=True)
torch.cuda.synchronize()
