"""Per-CTA timeline of the stream kernel (diagnostic build: `make -C paper_2002_03258_b200/csrc diag`).

  TSM2X_LIB_PATH_EXPERIMENT=paper_2002_03258_b200/libtsm2x_diag.so TSM2X_TC_DIAG=0 \
      python tools/timeline_probe.py [m=k] [n]

Each call (after a 252 MB read flush) prints one JSON line from the library on stderr: median and
max over CTAs, in us from the first CTA's entry, of: CTA entry, first TMA issue, first stage landed
in shared memory, producer done, consumers done."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2002_03258_b200 as tsm  # noqa: E402


def main():
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    k = int(sys.argv[3]) if len(sys.argv) > 3 else m
    A = tsm.colmajor_empty(m, k, torch.float64, "cuda")
    tsm.fill_uniform(A, 1)
    B = tsm.colmajor_empty(k, n, torch.float64, "cuda")
    tsm.fill_uniform(B, 2)
    C = tsm.colmajor_empty(m, n, torch.float64, "cuda")
    C.zero_()
    flush = torch.empty(63 << 20, dtype=torch.float32, device="cuda")
    red = torch.empty((), dtype=torch.float32, device="cuda")
    for i in range(6):
        torch.sum(flush, dim=0, out=red)
        torch.cuda.synchronize()
        print(f"call {i} m={m} k={k} n={n}", file=sys.stderr, flush=True)
        tsm.gemm(A, B, C, c_is_zero=(k <= 64), variant="l-opt2" if k <= 64 else "v3")
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
