"""Device-side gap between consecutive TSM2R calls (BASELINE configs[1], n=8): CUDA events right
before / after each stream-kernel launch (tsm2x_set_kernel_events) over back-to-back calls; prints
the mean kernel time and the mean gap from one kernel's end to the next one's start."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_03258_b200 as tsm  # noqa: E402
from paper_2002_03258_b200 import _lib  # noqa: E402

m = k = int(sys.argv[1]) if len(sys.argv) > 1 else 30720
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
det = len(sys.argv) > 4 and sys.argv[4] == "det"  # deterministic (chunk-ordered) combine
A = tsm.colmajor_empty(m, k, torch.float64, "cuda"); tsm.fill_uniform(A, 1)
B = tsm.colmajor_empty(k, n, torch.float64, "cuda"); tsm.fill_uniform(B, 2)
C = tsm.colmajor_empty(m, n, torch.float64, "cuda"); tsm.fill_uniform(C, 3)
lib = _lib.load()
s = torch.cuda.current_stream()
for _ in range(5):
    tsm.gemm(A, B, C, deterministic=det)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
for a, b in ev:
    a.record(s); b.record(s)
torch.cuda.synchronize()
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0.record(s)
for i in range(steps):
    lib.tsm2x_set_kernel_events(ctypes.c_void_p(ev[i][0].cuda_event), ctypes.c_void_p(ev[i][1].cuda_event))
    tsm.gemm(A, B, C, deterministic=det)
t1.record(s)
torch.cuda.synchronize()
kern = [a.elapsed_time(b) for a, b in ev]
gaps = [ev[i][1].elapsed_time(ev[i + 1][0]) for i in range(steps - 1)]
print(json.dumps({"m": m, "n": n, "deterministic": det, "env": {k: v for k, v in os.environ.items() if k.startswith("TSM2X")},
                  "ms_per_step": round(t0.elapsed_time(t1) / steps, 5), "kernel_ms": round(sum(kern) / steps, 5),
                  "gap_us": round(1000 * sum(gaps) / len(gaps), 2), "gap_us_max": round(1000 * max(gaps), 2)}))
