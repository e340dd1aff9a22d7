import sys, torch
sys.path.insert(0, ".")
import paper_2002_03258_b200 as tsm
mk = int(sys.argv[1]); n = int(sys.argv[2])
dt = torch.float64
A = tsm.colmajor_empty(mk, mk, dt, "cuda"); tsm.fill_uniform(A, 1)
B = tsm.colmajor_empty(mk, n, dt, "cuda"); tsm.fill_uniform(B, 2)
C = tsm.colmajor_empty(mk, n, dt, "cuda"); C.zero_()
for _ in range(6):
    tsm.gemm(A, B, C)
torch.cuda.synchronize()
