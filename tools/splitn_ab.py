"""A/B of the TSM2L split-n warp-shuffle kernel (csrc/tsm2l_splitn.cuh, impl "tsm2l-splitn")
against the production TSM2L path (impl "auto": the TMA stream kernel's single-chunk row blocks)
and the one-thread-per-row LDG kernel (impl "tsm2l"), on BASELINE configs[2] (fp64 2^24 x 16 x 16,
L_OPT2 zero C) and neighbours. Per impl: median device time per call over blocks of back-to-back
calls (sustained, A = 2 GB streams from HBM every call), and GB/s of the algorithmic bytes.
Prints JSON lines; python tools/splitn_ab.py > profiles/splitn_r02.json"""

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2002_03258_b200 as tsm  # noqa: E402

SHAPES = [(1 << 24, 16, 16, torch.float64), (1 << 24, 16, 16, torch.float32), (1 << 24, 16, 8, torch.float64),
          (1 << 25, 8, 8, torch.float32), (1 << 24, 32, 16, torch.float64)]
IMPLS = ["auto", "tsm2l", "tsm2l-splitn"]


def per_call_ms(fn, calls=30, blocks=7):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(blocks):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(calls):
            fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / calls)
    return statistics.median(out)


def _shapes_from_argv():
    """Optional shapes on the command line: m,k,n,{f64|f32} ..."""
    out = []
    for a in sys.argv[1:]:
        m, k, n, d = a.split(",")
        out.append((int(m), int(k), int(n), torch.float64 if d == "f64" else torch.float32))
    return out or SHAPES


def main():
    shapes = _shapes_from_argv()
    print(json.dumps({"what": "TSM2L split-n warp-shuffle A/B (tools/splitn_ab.py); sustained per-call ms, "
                      "C = A*B under the zero-C contract (L_OPT2)"}))
    for m, k, n, dt in shapes:
        A = tsm.colmajor_empty(m, k, dt, "cuda")
        tsm.fill_uniform(A, seed=1)
        B = tsm.colmajor_empty(k, n, dt, "cuda")
        tsm.fill_uniform(B, seed=2)
        eb = A.element_size()
        byts = eb * (m * k + k * n + m * n)
        ref = (A.double() @ B.double())
        row = {"m": m, "k": k, "n": n, "dtype": str(dt).split(".")[1]}
        for impl in IMPLS:
            C = tsm.colmajor_empty(m, n, dt, "cuda")
            ms = per_call_ms(lambda: tsm.gemm(A, B, C, variant="l-opt2", c_is_zero=True, impl=impl))
            err = float(((C.double() - ref).norm() / ref.norm()).item())
            row[impl] = {"ms": round(ms, 4), "GBps": round(byts / ms / 1e6, 1), "rel_frob": err}
            del C
        best = min(IMPLS, key=lambda i: row[i]["ms"])
        row["best"] = best
        print(json.dumps(row), flush=True)
        del A, B, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
