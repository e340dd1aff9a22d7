"""Interleaved A/B timing of tuning candidates in one process (sustained, alternating blocks so power/clock
drift hits every candidate alike). Usage: python tools/abtest.py [rounds]"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2002_03258_b200 as tsm  # noqa: E402
from paper_2002_03258_b200 import tuning  # noqa: E402

T = tuning.Tuning
CASES = {
    "l16": ((1 << 24, 16, 16, torch.float64), [T(), T(consumer=2), T(consumer=1)]),
}


def block_ms(A, B, C, reps, czero=False):
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        tsm.gemm(A, B, C, variant="l-opt2" if czero else "v3", c_is_zero=czero)
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    out = {}
    for name, ((m, k, n, dt), cands) in CASES.items():
        A = tsm.colmajor_empty(m, k, dt, "cuda")
        tsm.fill_uniform(A, 1)
        B = tsm.colmajor_empty(k, n, dt, "cuda")
        tsm.fill_uniform(B, 2)
        C = tsm.colmajor_empty(m, n, dt, "cuda")
        C.zero_()
        for t in cands:  # warm every variant (and the power state)
            tuning.set_tuning(t)
            block_ms(A, B, C, 50, name == "l16")
        res = {i: [] for i in range(len(cands))}
        for r in range(rounds):
            order = list(range(len(cands)))
            if r % 2:
                order.reverse()
            for i in order:
                tuning.set_tuning(cands[i])
                res[i].append(block_ms(A, B, C, 100, name == "l16"))
        tuning.set_tuning(None)
        rows = []
        for i, t in enumerate(cands):
            v = sorted(res[i])
            rows.append({"tuning": t.__dict__, "median_ms": round(v[len(v) // 2], 4), "min_ms": round(v[0], 4)})
        out[name] = rows
        print(json.dumps({name: rows}), flush=True)
        del A, B, C
        torch.cuda.empty_cache()
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "abtest.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
