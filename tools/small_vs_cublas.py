"""Per-call device time of the TSM2R path vs cuBLAS (torch.addmm on the same column-major
operands) across problem sizes, each call replayed from a CUDA graph after an L2 flush (cold A).
Small and mid-size problems are latency-bound (launch, ring fill, item epilogues); this is the
yardstick for them. Usage: python tools/small_vs_cublas.py [sizes...]"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2002_03258_b200 as tsm  # noqa: E402


def graph_us(fn, flush, reps=30):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return sorted(ts)[len(ts) // 2]


def main():
    impls = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--impls=")]
    impls = impls[0].split(",") if impls else ["auto"]
    sizes = [int(x) for x in sys.argv[1:] if not x.startswith("--")] or [1024, 2048, 4096, 8192, 16384]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for dt, n in ((torch.float64, 8), (torch.float64, 16), (torch.float32, 16)):
        for mk in sizes:
            A = tsm.colmajor_empty(mk, mk, dt, "cuda")
            tsm.fill_uniform(A, 1)
            B = tsm.colmajor_empty(mk, n, dt, "cuda")
            tsm.fill_uniform(B, 2)
            C = tsm.colmajor_empty(mk, n, dt, "cuda")
            C.zero_()
            C2 = C.clone()
            ours = {i: graph_us(lambda: tsm.gemm(A, B, C, impl=i), flush) for i in impls}
            cublas = graph_us(lambda: C2.addmm_(A, B), flush)
            eb = A.element_size()
            byts = eb * (mk * mk + mk * n + 2 * mk * n)
            extra = {f"{i}_us": round(v, 1) for i, v in ours.items() if i != "auto"}
            best = ours.get("auto", min(ours.values()))
            print(json.dumps({"dtype": str(dt).split(".")[1], "m=k": mk, "n": n, "tsm2x_us": round(best, 1), **extra,
                              "cublas_us": round(cublas, 1), "speedup": round(cublas / best, 2),
                              "tsm2x_GBps": round(byts / best / 1e3, 1), "ideal_us_at_7300": round(byts / 7.3e12 * 1e6, 1)}),
                  flush=True)
            del A, B, C, C2


if __name__ == "__main__":
    main()
