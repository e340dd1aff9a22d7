"""Burst time across problem sizes (fp64 / fp32 TSM2R, n = 8 / 16): how close small problems get
to the read roofline (launch, ramp-up, tail and combine overheads). Usage: python tools/sizes.py"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2002_03258_b200 as tsm  # noqa: E402


def main():
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > L2: cold A every call
    for dt, n in ((torch.float64, 8), (torch.float64, 16), (torch.float32, 16)):
        for mk in (1024, 2048, 4096, 8192, 16384):
            A = tsm.colmajor_empty(mk, mk, dt, "cuda")
            tsm.fill_uniform(A, 1)
            B = tsm.colmajor_empty(mk, n, dt, "cuda")
            tsm.fill_uniform(B, 2)
            C = tsm.colmajor_empty(mk, n, dt, "cuda")
            C.zero_()
            for _ in range(5):
                tsm.gemm(A, B, C)
            ts = []
            for _ in range(20):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                tsm.gemm(A, B, C)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = sorted(ts)[len(ts) // 2]
            # the same call replayed from a CUDA graph: no host work between the events
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                tsm.gemm(A, B, C)
            torch.cuda.current_stream().wait_stream(s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                tsm.gemm(A, B, C)
            tg = []
            for _ in range(20):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                tg.append(e0.elapsed_time(e1))
            msg = sorted(tg)[len(tg) // 2]
            # host cost of one eager call (Python wrapper + C++ launch path)
            import time
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(50):
                tsm.gemm(A, B, C)
            th = (time.perf_counter() - t0) / 50
            torch.cuda.synchronize()
            eb = A.element_size()
            byts = eb * (mk * mk + mk * n + 2 * mk * n)
            print(json.dumps({"dtype": str(dt).split(".")[1], "m=k": mk, "n": n, "us": round(ms * 1e3, 1), "graph_us": round(msg * 1e3, 1),
                              "host_us_per_call": round(th * 1e6, 1),
                              "GBps": round(byts / ms / 1e6, 1), "ideal_us_at_7300": round(byts / 7.3e12 * 1e6, 1)}),
                  flush=True)
            del A, B, C


if __name__ == "__main__":
    main()
