timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_apps_gpu.py -m gpu -q -x -k "tc32 or config4 or consumer or fp32 or equal_split or golden" 2>&1 | tail -2
cat > /tmp/tc.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2002_03258_b200 as tsm
m = k = 32768; n = 16
A = tsm.colmajor_empty(m, k, torch.float32, "cuda"); tsm.fill_uniform(A, 1)
B = tsm.colmajor_empty(k, n, torch.float32, "cuda"); tsm.fill_uniform(B, 2)
C = tsm.colmajor_empty(m, n, torch.float32, "cuda"); tsm.fill_uniform(C, 3)
for i in range(6):
    tsm.gemm(A, B, C); torch.cuda.synchronize()
PY
TSM2X_LIB_PATH_EXPERIMENT=paper_2002_03258_b200/libtsm2x_diag.so TSM2X_TC_DIAG=0 python /tmp/tc.py 2>&1 | grep tc32_diag | tail -1
WL=tsm2r_fp32_n16 CANDS="base;TSM2X_LIB_PATH_EXPERIMENT=paper_2002_03258_b200/libtsm2x_cw8.so" bash tools/burst_ab.sh
