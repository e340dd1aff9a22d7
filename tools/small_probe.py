"""Where the time of a small TSM2R call goes (BASELINE configs[0]: 4096^2 fp64, n=8, 134 MB of A).

Per-call device time of CUDA-graph replays of tsm2x.gemm under three L2 preconditions — a
256 MB write flush (the L2 then holds dirty lines that must be written back while A streams in),
a 256 MB read flush (clean L2, A not resident), and no flush (back-to-back calls) — next to
the same preconditions for a read-only reference: torch's sum over A (one kernel reading the
same 134 MB), i.e. what one launch can stream at this size. Prints JSON lines.
Usage: python tools/small_probe.py [m=k] [n] [--impls=auto,...]"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2002_03258_b200 as tsm  # noqa: E402


def graph_us(fn, pre, reps=40):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    ts = []
    for _ in range(reps):
        if pre is not None:
            pre()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize() if pre is not None else None
        ts.append((e0, e1))
    torch.cuda.synchronize()
    us = sorted(a.elapsed_time(b) * 1e3 for a, b in ts)
    mid = us[len(us) // 4: len(us) - len(us) // 4]  # event timestamps are ~2 us granular here: average
    return sum(mid) / len(mid)                      # the middle half instead of taking the median


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    impls = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--impls=")]
    impls = impls[0].split(",") if impls else ["auto"]
    mk = int(args[0]) if args else 4096
    n = int(args[1]) if len(args) > 1 else 8
    dt = torch.float64
    A = tsm.colmajor_empty(mk, mk, dt, "cuda")
    tsm.fill_uniform(A, 1)
    B = tsm.colmajor_empty(mk, n, dt, "cuda")
    tsm.fill_uniform(B, 2)
    C = tsm.colmajor_empty(mk, n, dt, "cuda")
    C.zero_()
    out = torch.empty((), dtype=dt, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush_f = flush.view(torch.float32)
    red = torch.empty((), dtype=torch.float32, device="cuda")
    pres = {"write_flush": lambda: flush.zero_(), "read_flush": lambda: torch.sum(flush_f, dim=0, out=red), "none": None}
    byts = 8 * (mk * mk + mk * n + 2 * mk * n)
    for pname, pre in pres.items():
        row = {"m=k": mk, "n": n, "pre": pname, "env": {k: v for k, v in os.environ.items() if k.startswith("TSM2X_")}}
        for i in impls:
            row[f"tsm2x_{i}_us"] = round(graph_us(lambda: tsm.gemm(A, B, C, impl=i), pre), 2)
        row["torch_sum_A_us"] = round(graph_us(lambda: torch.sum(A, dim=(0, 1), out=out), pre), 2)
        row["empty_graph_us"] = round(graph_us(lambda: out.zero_(), pre), 2)  # one 1-thread kernel: the floor
        row["ideal_us_at_7300"] = round(byts / 7.3e12 * 1e6, 2)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
